"""Quick throughput probe of the grouped tcgen05 GEMM at layer shapes (dev tool)."""
import sys, ctypes as C
sys.path.insert(0, ".")
import torch
import os, functools
from tests.test_gpu_gemm import _run as _run0, _groups
import tests.test_gpu_gemm as TG
_knobs = (int(os.environ.get('POL', '0')) << 12) | (int(os.environ.get('RASTER', '0')) << 16)
TG.KINDS = {k: v | _knobs for k, v in TG.KINDS.items()}
_run = functools.partial(_run0, pair=os.environ.get('PAIR', '1') == '1', sync=False)

import threading
try:
    import pynvml
    pynvml.nvmlInit()
    _nv = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:
    _nv = None


def bench(fn, iters=30):
    """Mean ms per call, and the mean SM clock (MHz) sampled while the calls ran."""
    for _ in range(3): fn()
    torch.cuda.synchronize()
    clk, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            if _nv is not None:
                clk.append(pynvml.nvmlDeviceGetClockInfo(_nv, pynvml.NVML_CLOCK_SM))
            stop.wait(0.005)
    th = threading.Thread(target=sample); th.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    bench.mhz = sum(clk) / len(clk) if clk else float("nan")
    return s.elapsed_time(e) / iters

H, F, G, rows = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
counts = [rows] * G
rg, off, R = _groups(counts)
X = torch.randn(R, H, device="cuda").bfloat16()
W13 = (torch.randn(G, 2*F, H, device="cuda") / H**0.5).bfloat16()
W2 = (torch.randn(G, H, F, device="cuda") / F**0.5).bfloat16()
h = torch.empty(R, 2*F, device="cuda", dtype=torch.bfloat16); act = torch.empty(R, F, device="cuda", dtype=torch.bfloat16)
y = torch.empty(R, H, device="cuda", dtype=torch.bfloat16); dY = torch.randn(R, H, device="cuda").bfloat16()
dH = torch.empty(R, 2*F, device="cuda", dtype=torch.bfloat16); dX = torch.empty(R, H, device="cuda", dtype=torch.bfloat16)
gW2 = torch.empty(G, H, F, device="cuda"); gW13 = torch.empty(G, 2*F, H, device="cuda")
tests = {
 "gateup": (lambda: _run("gateup", G, rg, off, 0, 2*F, H, X, R, H, W13, H, 2*F, G, H, 2*F*H, h, 2*F, out2=act, ldo2=F), 2*R*H*2*F),
 "down": (lambda: _run("down", G, rg, off, 0, H, F, act, R, F, W2, F, H, G, F, H*F, y, H), 2*R*H*F),
 "down_dgrad": (lambda: _run("down_dgrad", G, rg, off, 0, F, H, dY, R, H, W2, F, H, G, F, H*F, dH, 2*F, aux=h, ld_aux=2*F), 2*R*H*F),
 "up_dgrad": (lambda: _run("up_dgrad", G, rg, off, 0, H, 2*F, dH, R, 2*F, W13, H, 2*F, G, H, 2*F*H, dX, H), 2*R*H*2*F),
 "wgrad_w2": (lambda: _run("wgrad", G, rg, off, H, F, 0, dY, R, H, act, F, R, 1, F, 0, gW2, F, ogs=H*F), 2*R*H*F),
 "wgrad_w13": (lambda: _run("wgrad", G, rg, off, 2*F, H, 0, dH, R, 2*F, X, H, R, 1, H, 0, gW13, H, ogs=2*F*H), 2*R*H*2*F),
}
if os.environ.get("PLAIN") == "1":  # same shapes as the SwiGLU kernels, plain bf16 epilogue
    dA = torch.empty(R, F, device="cuda", dtype=torch.bfloat16)
    tests["gateup_plain"] = (lambda: _run("down", G, rg, off, 0, 2*F, H, X, R, H, W13, H, 2*F, G, H, 2*F*H, h, 2*F), 2*R*H*2*F)
    tests["down_dgrad_plain"] = (lambda: _run("up_dgrad", G, rg, off, 0, F, H, dY, R, H, W2, F, H, G, F, H*F, dA, F), 2*R*H*F)
if os.environ.get("ONLY"):
    tests = {k: v for k, v in tests.items() if k in os.environ["ONLY"].split(",")}
STALLS = os.environ.get("STALLS") == "1"  # needs FSEP_LIB_NAME=<a -DFSEP_GEMM_STALLS build>


def stalls(reset=False):
    from paper_2602_11686_b200 import _lib
    out = (C.c_ulonglong * 8)()
    _lib.check(_lib.load().mp_fsep_debug_gemm_stalls(out, 1 if reset else 0))
    return list(out)


tot_ms = tot_fl = 0
for name, (fn, fl) in tests.items():
    if STALLS:
        torch.cuda.synchronize(); stalls(reset=True)
    ms = bench(fn)
    if STALLS:
        torch.cuda.synchronize()
        c = stalls()
        life = max(c[4], 1)  # MMA-warp lifetime summed over the leader CTAs
        print(f"  stalls {name}: mma wait operands {100*c[0]/life:5.1f}%  mma wait accumulator {100*c[1]/life:5.1f}%  "
              f"producer wait stage {100*c[2]/(2*life):5.1f}%  producer ready/wave {100*c[6]/(2*life):5.1f}%  "
              f"epilogue wait {100*c[3]/(16*life):5.1f}%  epilogue drain {100*c[5]/(16*life):5.1f}%")
    tot_ms += ms; tot_fl += fl
    eff = fl / (ms * 1e-3) / (148 * 8192 * bench.mhz * 1e6)
    print(f"{name:16s} {ms:8.3f} ms  {fl/ms/1e9:8.1f} TFLOP/s  sm {bench.mhz:6.0f} MHz  per-clock {100*eff:5.1f}%")
print(f"total {tot_ms:.3f} ms {tot_fl/tot_ms/1e9:.1f} TFLOP/s")
