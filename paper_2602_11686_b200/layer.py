"""FSEP MoE layer, Python side: a thin owner of an mp_fsep_layer handle.

All compute runs in libmoeplan_b200.so (hand-written sm_100a kernels); torch is
only used here to hold device tensors and streams.  There is no fallback: if the
library or a GPU is missing, construction raises.

Modes (mp_fsep_desc.virtual_ranks):
  * real     -- one process per GPU (torch.distributed launch), world = N; ranks
                exchange CUDA IPC handles once (connect()) and then move tokens,
                shards and gradients with peer loads/stores over NVLink.
  * virtual  -- all N ranks emulated on one GPU (correctness / tests); inputs
                and outputs hold the N ranks' [T, H] blocks concatenated.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from ._lib import FsepDesc, check, load, u8p, u64p
from .planner import Config, Planner


@dataclass
class LayerSpec:
    n_experts: int
    top_k: int
    hidden: int
    ffn: int
    max_tokens: int
    capacity: int
    world: int = 1
    rank: int = 0
    virtual: bool = False
    max_recv_rows: int = 0
    resident: bool = False  # MP_FSEP_FLAG_RESIDENT_EXPERTS: pure EP baseline (E == N*C, fixed layout)
    local_first: bool = False  # MP_FSEP_FLAG_LOCAL_FIRST: non-parity local-first token routing
    copy_engine: bool = False  # MP_FSEP_FLAG_COPY_ENGINE: virtual mode runs the real N>1 copy-engine transport
    defer_rs: bool = False  # MP_FSEP_FLAG_DEFER_RS: reduce-scatter completes under the previous layer's backward


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    assert t.is_contiguous()
    return C.c_void_p(t.data_ptr())


class FsepLayer:
    def __init__(self, spec: LayerSpec, device: Optional[int] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("FsepLayer needs a CUDA device (no CPU fallback)")
        self.lib = load()
        self.spec = spec
        self.device = torch.cuda.current_device() if device is None else device
        d = FsepDesc(spec.n_experts, spec.top_k, spec.hidden, spec.ffn, spec.max_tokens, spec.capacity, spec.world,
                     spec.rank, 1 if spec.virtual else 0,
                     (1 if spec.resident else 0) | (2 if spec.local_first else 0) | (4 if spec.copy_engine else 0)
                     | (8 if spec.defer_rs else 0),
                     spec.max_recv_rows)
        h = C.c_void_p()
        check(self.lib.mp_fsep_layer_create(C.byref(d), self.device, C.byref(h)))
        self._h = h
        self._planner = None
        self.local_ranks = spec.world if (spec.virtual or spec.world == 1) else 1

    # ------------------------------------------------------------ multi-GPU
    def ipc_handle(self) -> bytes:
        n = self.lib.mp_fsep_ipc_bytes()
        buf = (C.c_char * n)()
        check(self.lib.mp_fsep_layer_ipc_handle(self._h, buf, n))
        return bytes(buf)

    def connect(self, handles: list[bytes], nccl_id: Optional[bytes] = None) -> None:
        blob = b"".join(handles)
        buf = (C.c_char * len(blob)).from_buffer_copy(blob)
        nid = (C.c_char * len(nccl_id)).from_buffer_copy(nccl_id) if nccl_id else None
        check(self.lib.mp_fsep_layer_connect(self._h, buf, nid))

    def connect_torch_distributed(self) -> None:
        """Exchange IPC handles (and rank 0's NCCL unique id, used by the FSEP_COMM=nccl
        transport) with torch.distributed (any backend)."""
        import torch.distributed as dist
        mine = self.ipc_handle()
        out = [None] * dist.get_world_size()
        dist.all_gather_object(out, mine)
        nid = [None]
        if dist.get_rank() == 0:
            buf = (C.c_char * 128)()
            check(self.lib.mp_fsep_nccl_unique_id(buf, 128))
            nid[0] = bytes(buf)
        dist.broadcast_object_list(nid, src=0)
        self.connect(out, nid[0])

    # ------------------------------------------------------------ parameters
    def load_expert(self, e: int, w1: torch.Tensor, w3: torch.Tensor, w2: torch.Tensor, stream=None) -> None:
        for t in (w1, w3, w2):
            assert t.dtype == torch.bfloat16 and t.is_contiguous()
        check(self.lib.mp_fsep_layer_load_expert(self._h, e, _ptr(w1), _ptr(w3), _ptr(w2), _stream(stream)))

    def load_router(self, wg: torch.Tensor, stream=None) -> None:
        assert wg.dtype == torch.bfloat16 and wg.is_contiguous()
        check(self.lib.mp_fsep_layer_load_router(self._h, _ptr(wg), _stream(stream)))

    def set_layout(self, A: np.ndarray) -> None:
        A = np.ascontiguousarray(A, dtype=np.uint8)
        check(self.lib.mp_fsep_layer_set_layout(self._h, A.ctypes.data_as(u8p)))

    def attach_planner(self, config: Config, layer: int = 0) -> Planner:
        self._planner = Planner(config, self.spec.world, layer)
        check(self.lib.mp_fsep_layer_attach_planner(self._h, self._planner._h))
        return self._planner

    def chain(self, next_layer: Optional["FsepLayer"]) -> None:
        """Issue next_layer's shard restore after this layer's gate-up GEMM (PAPER Fig.5)."""
        check(self.lib.mp_fsep_layer_chain(self._h, next_layer._h if next_layer is not None else None))

    def detach_planner(self) -> None:
        check(self.lib.mp_fsep_layer_attach_planner(self._h, None))
        self._planner = None

    # ------------------------------------------------------------ step
    def forward(self, x: torch.Tensor, bias: Optional[torch.Tensor], n_tokens: int, y: torch.Tensor,
                stream=None) -> torch.Tensor:
        check(self.lib.mp_fsep_layer_forward(self._h, _ptr(x), _ptr(bias), n_tokens, _ptr(y), _stream(stream)))
        return y

    def backward(self, dy: torch.Tensor, dx: torch.Tensor, stream=None) -> torch.Tensor:
        check(self.lib.mp_fsep_layer_backward(self._h, _ptr(dy), _ptr(dx), _stream(stream)))
        return dx

    def graph_step(self, x, bias, n_tokens, y, dy, dx, stream=None) -> None:
        check(self.lib.mp_fsep_layer_graph_step(self._h, _ptr(x), _ptr(bias), n_tokens, _ptr(y), _ptr(dy), _ptr(dx),
                                                _stream(stream)))

    # ------------------------------------------------------------ outputs
    def histogram(self) -> np.ndarray:
        R = np.zeros((self.spec.world, self.spec.n_experts), dtype=np.uint64)
        check(self.lib.mp_fsep_layer_histogram(self._h, R.ctypes.data_as(u64p)))
        return R

    def expert_grad(self, e: int, stream=None):
        s = self.spec
        dw1 = torch.zeros(s.ffn, s.hidden, device="cuda", dtype=torch.float32)
        dw3 = torch.zeros_like(dw1)
        dw2 = torch.zeros(s.hidden, s.ffn, device="cuda", dtype=torch.float32)
        check(self.lib.mp_fsep_layer_expert_grad(self._h, e, _ptr(dw1), _ptr(dw3), _ptr(dw2), _stream(stream)))
        return dw1, dw3, dw2

    def router_grad(self, vrank: int = 0) -> torch.Tensor:
        s = self.spec
        out = torch.empty(s.n_experts, s.hidden, device="cuda", dtype=torch.float32)
        check(self.lib.mp_fsep_layer_router_grad(self._h, vrank, _ptr(out), _stream(None)))
        return out

    def read(self, name: str, vrank: int = 0) -> np.ndarray:
        need = C.c_uint64()
        check(self.lib.mp_fsep_layer_read(self._h, name.encode(), vrank, None, 0, C.byref(need)))
        buf = np.empty(need.value, dtype=np.uint8)
        check(self.lib.mp_fsep_layer_read(self._h, name.encode(), vrank, buf.ctypes.data_as(C.c_void_p),
                                          need.value, None))
        return buf

    def stats(self):
        n = C.c_uint64()
        ms, fl = C.c_double(), C.c_double()
        check(self.lib.mp_fsep_layer_stats(self._h, C.byref(n), C.byref(ms), C.byref(fl)))
        return {"kernel_launches": n.value, "gemm_ms": ms.value, "gemm_flops": fl.value}

    PHASES = ["param_barrier", "router_scan", "R_barrier", "plan", "dispatch", "dispatch_barrier", "restore_wait",
              "fwd_gemm_gateup", "fwd_gemm_down", "fwd_barrier", "combine", "combine_bwd_router_wgrad", "bwd_barrier0", "bwd_gemms",
              "rs_push_wait", "rs_barrier", "rs_sum", "unpermute", "grad_reduce_scatter_kernel", "step_total", "restore_start",
              "restore_ms", "layout_h2d", "gap_between_steps", "host_planner_wait", "hist_on_host_at", "planner_done_at", "restore_landed_ms"]

    def phase_ms(self):
        """Mean per-phase device times (needs FSEP_PHASE_TIMING=1 at layer creation), or None."""
        out = (C.c_double * len(self.PHASES))()
        if self.lib.mp_fsep_layer_phase_ms(self._h, out, len(self.PHASES)) != 0:
            return None
        return {k: round(out[i], 4) for i, k in enumerate(self.PHASES)}

    def check(self) -> int:
        """Synchronise and report device-detected failures of the steps so far
        (raises MoeplanError, status MP_ERR_DEVICE, if any; returns 0 otherwise)."""
        bits = C.c_uint32()
        st = self.lib.mp_fsep_layer_check(self._h, C.byref(bits))
        self.last_error_bits = bits.value
        check(st)
        return bits.value

    def debug_restore_ms(self, iters: int = 10) -> float:
        ms = C.c_double()
        check(self.lib.mp_fsep_layer_debug_restore(self._h, iters, C.byref(ms)))
        return ms.value

    def debug_inject(self, what: str) -> None:
        check(self.lib.mp_fsep_layer_debug_inject(self._h, what.encode()))

    def stats_reset(self) -> None:
        check(self.lib.mp_fsep_layer_stats_reset(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            if self._planner is not None:
                self.lib.mp_fsep_layer_attach_planner(self._h, None)
            self.lib.mp_fsep_layer_chain(self._h, None)
            self.lib.mp_fsep_layer_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
