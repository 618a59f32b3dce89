"""ctypes binding of libmoeplan_b200.so (the product C ABI: include/moeplan.h +
include/moeplan_fsep.h).  Loading fails loudly -- there is no Python or CPU
fallback for anything behind this boundary."""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

_LOCK = threading.Lock()
_LIB = None

MP_STATUS = {0: "ok", 1: "invalid_argument", 2: "parse", 3: "io", 4: "infeasible",
             5: "budget_exceeded", 6: "internal", 7: "device"}


class MoeplanError(RuntimeError):
    """A non-OK mp_status; .status is the code, .kind its name (moeplan.h:33-42)."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = MP_STATUS.get(status, "unknown")
        super().__init__(f"{self.kind}: {message}")


u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
dblp = C.POINTER(C.c_double)
vp = C.c_void_p
cp = C.c_char_p
u32 = C.c_uint32
u64 = C.c_uint64


class FsepDesc(C.Structure):
    _fields_ = [("n_experts", u32), ("top_k", u32), ("hidden", u32), ("ffn", u32),
                ("max_tokens", u32), ("capacity", u32), ("world", u32), ("rank", u32),
                ("virtual_ranks", u32), ("flags", u32), ("max_recv_rows", u64)]


_SIGS = {
    # moeplan.h
    "mp_status_name": (cp, [C.c_int]),
    "mp_last_error": (cp, []),
    "mp_string_free": (None, [vp]),
    "mp_trace_generate": (C.c_int, [cp, u64p, C.POINTER(vp)]),
    "mp_trace_load": (C.c_int, [cp, C.POINTER(vp)]),
    "mp_trace_save": (C.c_int, [vp, cp]),
    "mp_trace_dims": (C.c_int, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]),
    "mp_trace_layer_count": (C.c_int, [vp, C.POINTER(u32)]),
    "mp_trace_layer_at": (C.c_int, [vp, u32, C.POINTER(u32)]),
    "mp_trace_stats_json": (C.c_int, [vp, C.POINTER(vp)]),
    "mp_trace_free": (None, [vp]),
    "mp_config_parse": (C.c_int, [cp, C.POINTER(vp)]),
    "mp_config_load": (C.c_int, [cp, C.POINTER(vp)]),
    "mp_config_set_seed": (C.c_int, [vp, u64]),
    "mp_config_trace_path": (cp, [vp]),
    "mp_config_out_path": (cp, [vp]),
    "mp_config_free": (None, [vp]),
    "mp_plan_layer_json": (C.c_int, [vp, vp, u32, C.POINTER(vp)]),
    "mp_simulate": (C.c_int, [vp, vp, cp, C.POINTER(vp), C.POINTER(vp)]),
    "mp_analyze_json": (C.c_int, [vp, C.POINTER(vp)]),
    "mp_oracle_gap_json": (C.c_int, [vp, cp, C.POINTER(vp)]),
    # moeplan_fsep.h -- planner arrays
    "mp_fsep_planner_create": (C.c_int, [vp, u32, u32, C.POINTER(vp)]),
    "mp_fsep_planner_observe": (C.c_int, [vp, u64p]),
    "mp_fsep_planner_next": (C.c_int, [vp, u8p]),
    "mp_fsep_planner_free": (None, [vp]),
    "mp_fsep_plan_next": (C.c_int, [vp, u64p, u32, u32, u8p]),
    "mp_fsep_plan_layout": (C.c_int, [u32, u32, u32, C.c_double, C.c_double, C.c_double, C.c_double,
                                      u32, u64, u64p, u8p]),
    "mp_fsep_lite_routing": (C.c_int, [u32, u32, u64p, u8p, u64p]),
    "mp_fsep_static_layout": (C.c_int, [u32, u32, u32, u8p]),
    "mp_fsep_even_layout": (C.c_int, [u32, u32, u32, u8p]),
    "mp_fsep_time_cost": (C.c_int, [u32, u32, u64p, u8p, C.c_double, C.c_double, C.c_double, C.c_double,
                                    dblp, dblp, dblp, u64p]),
    "mp_fsep_trace_popularity": (C.c_int, [cp, dblp, u64]),
    "mp_fsep_trace_create": (C.c_int, [u32, u32, C.POINTER(vp)]),
    "mp_fsep_trace_append": (C.c_int, [vp, u32, u32, u64p]),
    # moeplan_fsep.h -- GPU layer
    "mp_fsep_layer_create": (C.c_int, [C.POINTER(FsepDesc), C.c_int, C.POINTER(vp)]),
    "mp_fsep_layer_free": (None, [vp]),
    "mp_fsep_ipc_bytes": (C.c_size_t, []),
    "mp_fsep_nccl_unique_id": (C.c_int, [vp, C.c_size_t]),
    "mp_fsep_layer_ipc_handle": (C.c_int, [vp, vp, C.c_size_t]),
    "mp_fsep_layer_connect": (C.c_int, [vp, vp, vp]),
    "mp_fsep_layer_connect_local": (C.c_int, [C.POINTER(vp), u32]),
    "mp_fsep_layer_load_expert": (C.c_int, [vp, u32, vp, vp, vp, vp]),
    "mp_fsep_layer_load_router": (C.c_int, [vp, vp, vp]),
    "mp_fsep_layer_set_layout": (C.c_int, [vp, u8p]),
    "mp_fsep_layer_attach_planner": (C.c_int, [vp, vp]),
    "mp_fsep_layer_chain": (C.c_int, [vp, vp]),
    "mp_fsep_layer_forward": (C.c_int, [vp, vp, vp, u32, vp, vp]),
    "mp_fsep_layer_backward": (C.c_int, [vp, vp, vp, vp]),
    "mp_fsep_layer_histogram": (C.c_int, [vp, u64p]),
    "mp_fsep_layer_expert_grad": (C.c_int, [vp, u32, vp, vp, vp, vp]),
    "mp_fsep_layer_router_grad": (C.c_int, [vp, u32, vp, vp]),
    "mp_fsep_layer_read": (C.c_int, [vp, cp, u32, vp, u64, u64p]),
    "mp_fsep_layer_stats": (C.c_int, [vp, u64p, dblp, dblp]),
    "mp_fsep_layer_stats_reset": (C.c_int, [vp]),
    "mp_fsep_layer_phase_ms": (C.c_int, [vp, dblp, u32]),
    "mp_fsep_layer_graph_step": (C.c_int, [vp, vp, vp, u32, vp, vp, vp, vp]),
    "mp_fsep_layer_check": (C.c_int, [vp, C.POINTER(u32)]),
    "mp_fsep_layer_debug_inject": (C.c_int, [vp, cp]),
    "mp_fsep_layer_debug_restore": (C.c_int, [vp, C.c_int, dblp]),
}


def lib_path() -> Path:
    from .build import lib_path as _p
    return _p()


def load():
    """Load (never build) the product library.  Raises if it is missing."""
    global _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        path = lib_path()
        if not path.exists():
            raise RuntimeError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the FSEP path has no fallback)")
        lib = C.CDLL(str(path), mode=C.RTLD_LOCAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue  # reported by missing_symbols(); calling it raises AttributeError
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
        return lib


def exported_symbols():
    return list(_SIGS)


def missing_symbols():
    lib = load()
    return [n for n in _SIGS if getattr(lib, n, None) is None]


def check(status: int) -> None:
    if status != 0:
        raise MoeplanError(status, load().mp_last_error().decode())


def take_string(ptr: C.c_void_p) -> str:
    """Copy and free a malloc'd string returned through the ABI."""
    if not ptr:
        return ""
    lib = load()
    text = C.cast(ptr, C.c_char_p).value.decode()
    lib.mp_string_free(ptr)
    return text
