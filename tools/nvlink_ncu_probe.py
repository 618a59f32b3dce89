"""NVLink bytes of the layer step's own kernels, from ncu's NVLink counters (dev tool).

ncu must not profile multi-process (multi-rank) runs, and the pool's driver reports
nvidia-smi's NVLink throughput counters as N/A.  This probe drives a real-mode N-rank
layer from ONE process (mp_fsep_layer_connect_local: direct peer access instead of
CUDA IPC), so ncu can profile rank 0's kernels:

  FSEP_SPIN_TIMEOUT_MS=200 ncu --devices 0 --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum \
      -k regex:"dispatch_tma|combine_bwd|grouped_gemm_pair" python tools/nvlink_ncu_probe.py mixtral 2

Under ncu the launches are serialised, so the cross-GPU barriers time out (bounded,
reported, ignored here); the data movement of each profiled kernel is unchanged.
Without ncu the probe checks the step is healthy (no device-detected failure).
usage: python tools/nvlink_ncu_probe.py {mixtral|fine} N [steps]"""
import ctypes as C
import os
import sys
from pathlib import Path

# One host thread drives every GPU: with lazy module loading the first launch of a kernel
# on a device waits for that device to go idle, which a cross-GPU barrier kernel waiting
# for a not-yet-launched peer never does -- load every module up front instead.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import layer_oracle as LO  # noqa: E402  (routing bias generator only)
from paper_2602_11686_b200._lib import check, load  # noqa: E402
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec  # noqa: E402

cfgs = {"mixtral": (8, 2, 4096, 14336, 16384), "fine": (64, 8, 2048, 1408, 32768)}
E, K, H, F, T = cfgs[sys.argv[1]]
N = int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
C_ = max(K, min(E, 2 * E // N))
layers, io, streams = [], [], []
for r in range(N):
    torch.cuda.set_device(r)
    L = FsepLayer(LayerSpec(E, K, H, F, T, C_, world=N, rank=r), device=r)
    g = torch.Generator(device=f"cuda:{r}").manual_seed(7)
    for e in range(E):
        L.load_expert(e, (torch.randn(F, H, device=f"cuda:{r}", generator=g) / H ** 0.5).bfloat16(),
                      (torch.randn(F, H, device=f"cuda:{r}", generator=g) / H ** 0.5).bfloat16(),
                      (torch.randn(H, F, device=f"cuda:{r}", generator=g) / F ** 0.5).bfloat16())
    L.load_router((torch.randn(E, H, device=f"cuda:{r}", generator=g) * 0.02).bfloat16())
    rng = np.random.default_rng(r)
    x = torch.randn(T, H, device=f"cuda:{r}", generator=g).bfloat16()
    io.append(dict(x=x, dy=(torch.randn(T, H, device=f"cuda:{r}", generator=g) * 0.1).bfloat16(),
                   bias=torch.from_numpy(LO.make_bias(rng, T, E, 1.2, np.random.default_rng(5).permutation(E))).to(f"cuda:{r}"),
                   y=torch.empty_like(x), dx=torch.empty_like(x)))
    streams.append(torch.cuda.Stream(device=r))
    layers.append(L)
    torch.cuda.synchronize(r)
handles = (C.c_void_p * N)(*[L._h.value for L in layers])
check(load().mp_fsep_layer_connect_local(handles, N))
for _ in range(steps):
    # under ncu the serialised launches time the cross-GPU waits out; drop those reports
    # (no device sync) so every call of the step is issued -- a no-op in a plain run
    for r, L in enumerate(layers):
        with torch.cuda.device(r):
            L.debug_inject("clear_errors")
            L.forward(io[r]["x"], io[r]["bias"], T, io[r]["y"], stream=streams[r])
    for r, L in enumerate(layers):
        with torch.cuda.device(r):
            L.debug_inject("clear_errors")
            L.backward(io[r]["dy"], io[r]["dx"], stream=streams[r])
for r in range(N):
    torch.cuda.synchronize(r)
status = []
for r, L in enumerate(layers):
    with torch.cuda.device(r):
        try:
            L.check()
            status.append("ok")
        except Exception as exc:  # expected under ncu (serialised launches time out the barriers)
            status.append(str(exc)[:90])
print("nvlink probe", sys.argv[1], "N", N, "C", C_, "status", status, flush=True)
for L in layers:
    L.close()
