"""Host planner, Python side: a thin mirror of the C ABI (include/moeplan.h,
include/moeplan_fsep.h).  Every call goes through libmoeplan_b200.so -- the C++
planner that reproduces /root/reference/proj/src/planner.cpp bit for bit.

Names follow the reference: Config/Trace handles (moeplan.h:43-87),
plan_layer_json / simulate / analyze (moeplan.h:89-107), and the array-level
plan_layout / lite_routing / static_ep_layout / even_replication_layout
(planner.hpp:32-100) on numpy arrays R[N,E] uint64, A[E,N] uint8, S[N,E,N].
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from ._lib import check, load, take_string, u8p, u64p


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(u64p)


def _p8(a: np.ndarray):
    return a.ctypes.data_as(u8p)


class Config:
    """mp_config handle (moeplan.h:78-87)."""

    def __init__(self, text: Optional[str] = None, path: Optional[str] = None):
        lib = load()
        h = C.c_void_p()
        if text is not None:
            check(lib.mp_config_parse(text.encode(), C.byref(h)))
        else:
            check(lib.mp_config_load(str(path).encode(), C.byref(h)))
        self._h = h

    def set_seed(self, seed: int) -> None:
        check(load().mp_config_set_seed(self._h, seed))

    @property
    def trace_path(self) -> str:
        return load().mp_config_trace_path(self._h).decode()

    @property
    def out_path(self) -> str:
        return load().mp_config_out_path(self._h).decode()

    def __del__(self):
        if getattr(self, "_h", None):
            load().mp_config_free(self._h)
            self._h = None


class Trace:
    """mp_trace handle (moeplan.h:54-74)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def generate(cls, spec_json: str, seed: Optional[int] = None) -> "Trace":
        h = C.c_void_p()
        s = C.c_uint64(seed) if seed is not None else None
        check(load().mp_trace_generate(spec_json.encode(), C.byref(s) if s is not None else None, C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "Trace":
        h = C.c_void_p()
        check(load().mp_trace_load(str(path).encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def create(cls, n_devices: int, n_experts: int) -> "Trace":
        """Empty trace to record observed histograms (mp_fsep_trace_create)."""
        h = C.c_void_p()
        check(load().mp_fsep_trace_create(n_devices, n_experts, C.byref(h)))
        return cls(h)

    def append(self, iteration: int, layer: int, R) -> None:
        R = _u64(R)
        check(load().mp_fsep_trace_append(self._h, iteration, layer, _p64(R)))

    def save(self, path: str) -> None:
        check(load().mp_trace_save(self._h, str(path).encode()))

    def dims(self):
        n, e, r = C.c_uint32(), C.c_uint32(), C.c_uint32()
        check(load().mp_trace_dims(self._h, C.byref(n), C.byref(e), C.byref(r)))
        return n.value, e.value, r.value

    def layers(self):
        lib = load()
        cnt = C.c_uint32()
        check(lib.mp_trace_layer_count(self._h, C.byref(cnt)))
        out = []
        for i in range(cnt.value):
            v = C.c_uint32()
            check(lib.mp_trace_layer_at(self._h, i, C.byref(v)))
            out.append(v.value)
        return out

    def stats_json(self) -> str:
        p = C.c_void_p()
        check(load().mp_trace_stats_json(self._h, C.byref(p)))
        return take_string(p)

    def __del__(self):
        if getattr(self, "_h", None):
            load().mp_trace_free(self._h)
            self._h = None


def plan_layer_json(config: Config, trace: Trace, layer: int) -> str:
    p = C.c_void_p()
    check(load().mp_plan_layer_json(config._h, trace._h, layer, C.byref(p)))
    return take_string(p)


def simulate(config: Config, trace: Trace, schedulers: str = "laer,static_ep"):
    rj, rc = C.c_void_p(), C.c_void_p()
    check(load().mp_simulate(config._h, trace._h, schedulers.encode(), C.byref(rj), C.byref(rc)))
    return take_string(rj), take_string(rc)


def oracle_gap_json(config: Config, instance_json: str) -> str:
    """mp_oracle_gap_json: greedy planner vs the exact optimum on one tiny instance."""
    p = C.c_void_p()
    check(load().mp_oracle_gap_json(config._h, instance_json.encode(), C.byref(p)))
    return take_string(p)


def analyze_json(config: Config) -> str:
    p = C.c_void_p()
    check(load().mp_analyze_json(config._h, C.byref(p)))
    return take_string(p)


# ---------------------------------------------------------------- arrays

def plan_layout(R, capacity: int, *, bandwidth: float = 900e9, v_comm: float = 8192.0,
                v_comp: float = 3.52e8, b_comp: float = 1.6354e15, epsilon: int = 2, seed: int = 0) -> np.ndarray:
    """plan_layout on history [R] with Topology(1, N, bw, bw) (planner.cpp:369-414). Returns A[E,N]."""
    R = _u64(R)
    n, e = R.shape
    A = np.zeros((e, n), dtype=np.uint8)
    check(load().mp_fsep_plan_layout(n, e, capacity, bandwidth, v_comm, v_comp, b_comp, epsilon, seed,
                                     _p64(R), _p8(A)))
    return A


def lite_routing(R, A) -> np.ndarray:
    """Dense S[src, expert, dst] of lite_routing (planner.cpp:238-287), single-node topology."""
    R, A = _u64(R), _u8(A)
    n, e = R.shape
    S = np.zeros((n, e, n), dtype=np.uint64)
    check(load().mp_fsep_lite_routing(n, e, _p64(R), _p8(A), _p64(S)))
    return S


def static_ep_layout(n_devices: int, n_experts: int, capacity: int) -> np.ndarray:
    A = np.zeros((n_experts, n_devices), dtype=np.uint8)
    check(load().mp_fsep_static_layout(n_devices, n_experts, capacity, _p8(A)))
    return A


def even_replication_layout(n_devices: int, n_experts: int, capacity: int) -> np.ndarray:
    A = np.zeros((n_experts, n_devices), dtype=np.uint8)
    check(load().mp_fsep_even_layout(n_devices, n_experts, capacity, _p8(A)))
    return A


def time_cost(R, A, *, bandwidth: float, v_comm: float, v_comp: float, b_comp: float):
    R, A = _u64(R), _u8(A)
    n, e = R.shape
    out = [C.c_double(), C.c_double(), C.c_double()]
    mr = C.c_uint64()
    check(load().mp_fsep_time_cost(n, e, _p64(R), _p8(A), bandwidth, v_comm, v_comp, b_comp,
                                   *[C.byref(o) for o in out], C.byref(mr)))
    return {"t_comm": out[0].value, "t_comp": out[1].value, "t_total": out[2].value, "max_recv": mr.value}


def trace_popularity(spec_json: str) -> np.ndarray:
    """[layers, iterations, experts] popularity of the drifting synthetic trace (generate_trace)."""
    import json as _json
    spec = _json.loads(spec_json)
    shape = (spec.get("n_layers", 1), spec["n_iterations"], spec["n_experts"])
    out = np.zeros(shape, dtype=np.float64)
    check(load().mp_fsep_trace_popularity(spec_json.encode(), out.ctypes.data_as(C.POINTER(C.c_double)), out.size))
    return out


def plan_next(config: Config, R, layer: int = 0) -> np.ndarray:
    """mp_fsep_plan_next: next-step layout of MoE layer `layer` from one observed R."""
    R = _u64(R)
    n, e = R.shape
    A = np.zeros((e, n), dtype=np.uint8)
    check(load().mp_fsep_plan_next(config._h, _p64(R), n, layer, _p8(A)))
    return A


class Planner:
    """Per-layer planner with history and the runtime's one-step lag
    (sim.cpp:99-149): next() is even_replication_layout before any observation,
    then plan_layout(history)."""

    def __init__(self, config: Config, n_devices: int, layer: int = 0):
        self._cfg = config  # keep alive
        h = C.c_void_p()
        check(load().mp_fsep_planner_create(config._h, n_devices, layer, C.byref(h)))
        self._h = h
        self.n_devices = n_devices

    def observe(self, R) -> None:
        R = _u64(R)
        check(load().mp_fsep_planner_observe(self._h, _p64(R)))

    def next(self, n_experts: int) -> np.ndarray:
        A = np.zeros((n_experts, self.n_devices), dtype=np.uint8)
        check(load().mp_fsep_planner_next(self._h, _p8(A)))
        return A

    def __del__(self):
        if getattr(self, "_h", None):
            load().mp_fsep_planner_free(self._h)
            self._h = None
