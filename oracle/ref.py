"""ORACLE (test infrastructure only): ctypes binding of the UNMODIFIED reference
library built by oracle/build_ref.sh into oracle/_ref/libmoeplan_ref.so, through
the reference's own C ABI (/root/reference/proj/include/moeplan.h:46-107), plus
the refplan_bench timing driver (oracle/refplan_bench.cpp).

Available wherever oracle/_ref was built (this container; it also travels to the
GPU box with the repo snapshot).  Callers must treat absence as "skip", never as
a reason to fall back to something else.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
REF_LIB = REF_DIR / "libmoeplan_ref.so"
REF_BENCH = REF_DIR / "refplan_bench"
REFERENCE_SRC = Path(os.environ.get("MOEPLAN_REFERENCE", "/root/reference/proj"))

_lib = None


def ensure_built() -> bool:
    """Build oracle/_ref from the reference sources if they are present here."""
    if REF_LIB.exists() and REF_BENCH.exists():
        return True
    if not (REFERENCE_SRC / "src").is_dir():
        return False
    subprocess.run(["bash", str(HERE / "build_ref.sh")], check=True, stdout=subprocess.DEVNULL)
    return REF_LIB.exists()


def available() -> bool:
    return REF_LIB.exists() or ensure_built()


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError("reference oracle library not built (oracle/_ref)")
        L = C.CDLL(str(REF_LIB), mode=C.RTLD_LOCAL)
        vp, cp, u32, u64 = C.c_void_p, C.c_char_p, C.c_uint32, C.c_uint64
        sigs = {
            "mp_last_error": (cp, []),
            "mp_string_free": (None, [vp]),
            "mp_trace_generate": (C.c_int, [cp, C.POINTER(u64), C.POINTER(vp)]),
            "mp_trace_load": (C.c_int, [cp, C.POINTER(vp)]),
            "mp_trace_free": (None, [vp]),
            "mp_trace_stats_json": (C.c_int, [vp, C.POINTER(vp)]),
            "mp_config_parse": (C.c_int, [cp, C.POINTER(vp)]),
            "mp_config_free": (None, [vp]),
            "mp_plan_layer_json": (C.c_int, [vp, vp, u32, C.POINTER(vp)]),
            "mp_simulate": (C.c_int, [vp, vp, cp, C.POINTER(vp), C.POINTER(vp)]),
            "mp_analyze_json": (C.c_int, [vp, C.POINTER(vp)]),
            "mp_oracle_gap_json": (C.c_int, [vp, cp, C.POINTER(vp)]),
        }
        for n, (r, a) in sigs.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def _check(st: int):
    if st != 0:
        raise RefError(st, lib().mp_last_error().decode())


def _take(p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    lib().mp_string_free(p)
    return s


class _Handle:
    def __init__(self, h, free):
        self.h, self._free = h, free

    def __del__(self):
        if self.h:
            self._free(self.h)


def config(text: str) -> _Handle:
    h = C.c_void_p()
    _check(lib().mp_config_parse(text.encode(), C.byref(h)))
    return _Handle(h, lib().mp_config_free)


def trace_generate(spec_json: str) -> _Handle:
    h = C.c_void_p()
    _check(lib().mp_trace_generate(spec_json.encode(), None, C.byref(h)))
    return _Handle(h, lib().mp_trace_free)


def trace_load(path: str) -> _Handle:
    h = C.c_void_p()
    _check(lib().mp_trace_load(str(path).encode(), C.byref(h)))
    return _Handle(h, lib().mp_trace_free)


def plan_layer_json(cfg: _Handle, trace: _Handle, layer: int) -> str:
    p = C.c_void_p()
    _check(lib().mp_plan_layer_json(cfg.h, trace.h, layer, C.byref(p)))
    return _take(p)


def simulate(cfg: _Handle, trace: _Handle, schedulers: str):
    a, b = C.c_void_p(), C.c_void_p()
    _check(lib().mp_simulate(cfg.h, trace.h, schedulers.encode(), C.byref(a), C.byref(b)))
    return _take(a), _take(b)


def oracle_gap_json(cfg: _Handle, instance_json: str) -> str:
    out = C.c_void_p()
    _check(lib().mp_oracle_gap_json(cfg.h, instance_json.encode(), C.byref(out)))
    return _take(out)


def analyze_json(cfg: _Handle) -> str:
    p = C.c_void_p()
    _check(lib().mp_analyze_json(cfg.h, C.byref(p)))
    return _take(p)


def stats_json(trace: _Handle) -> str:
    p = C.c_void_p()
    _check(lib().mp_trace_stats_json(trace.h, C.byref(p)))
    return _take(p)


def plan_bench(R, capacity: int, iters: int, *, bandwidth: float, v_comm: float, v_comp: float,
               b_comp: float, seed: int = 0) -> dict:
    """Time reference plan_layout + lite_routing on R (1 core) via refplan_bench."""
    if not available():
        raise FileNotFoundError("reference oracle not built")
    n, e = len(R), len(R[0])
    text = "\n".join(" ".join(str(int(v)) for v in row) for row in R)
    out = subprocess.run([str(REF_BENCH), str(n), str(e), str(capacity), str(iters), repr(float(bandwidth)),
                          repr(float(v_comm)), repr(float(v_comp)), repr(float(b_comp)), str(seed)],
                         input=text, capture_output=True, text=True, check=True)
    return json.loads(out.stdout)
