"""Interleaved A/B of grouped-GEMM variants at layer shapes (dev tool, GPU box).

Each variant is a per-call policy word (GemmParams::policy bits / raster), so the
variants alternate inside one process: rounds x (variant A for ~T s, variant B ...),
reporting mean ms per call, the mean SM clock sampled every 2 ms during the run, and
kilocycles per call (ms x MHz), which is what a kernel change should move when the
board's power cap sets the clock.

usage: python tools/gemm_ab.py H F G rows GEMM "name=policy[:raster]" ... [--rounds R] [--secs S]
GEMM in gateup, down, down_dgrad, up_dgrad, wgrad_w2, wgrad_w13."""
import argparse
import ctypes as C
import sys
import threading
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import tests.test_gpu_gemm as TG  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("H", type=int)
ap.add_argument("F", type=int)
ap.add_argument("G", type=int)
ap.add_argument("rows", type=str, help="rows per group, or comma list")
ap.add_argument("gemm")
ap.add_argument("variants", nargs="+")
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--secs", type=float, default=1.5)
a = ap.parse_args()
H, F, G = a.H, a.F, a.G
counts = [int(x) for x in a.rows.split(",")] if "," in a.rows else [int(a.rows)] * G
rg, off, R = TG._groups(counts)
X = torch.randn(R, H, device="cuda").bfloat16()
W13 = (torch.randn(G, 2 * F, H, device="cuda") / H ** 0.5).bfloat16()
W2 = (torch.randn(G, H, F, device="cuda") / F ** 0.5).bfloat16()
h = torch.randn(R, 2 * F, device="cuda").bfloat16()
act = torch.empty(R, F, device="cuda", dtype=torch.bfloat16)
y = torch.empty(R, H, device="cuda", dtype=torch.bfloat16)
dY = torch.randn(R, H, device="cuda").bfloat16()
dH = torch.empty(R, 2 * F, device="cuda", dtype=torch.bfloat16)
dX = torch.empty(R, H, device="cuda", dtype=torch.bfloat16)
gW2 = torch.empty(G, H, F, device="cuda")
gW13 = torch.empty(G, 2 * F, H, device="cuda")


def call(kind_bits):
    TG.KINDS = {k: v | kind_bits for k, v in {"gateup": 0, "down": 1, "down_dgrad": 2, "up_dgrad": 3, "wgrad": 4}.items()}
    r = lambda *args, **kw: TG._run(*args, sync=False, **kw)
    return {
        "gateup": lambda: r("gateup", G, rg, off, 0, 2 * F, H, X, R, H, W13, H, 2 * F, G, H, 2 * F * H, h, 2 * F, out2=act, ldo2=F),
        "down": lambda: r("down", G, rg, off, 0, H, F, act, R, F, W2, F, H, G, F, H * F, y, H),
        "down_dgrad": lambda: r("down_dgrad", G, rg, off, 0, F, H, dY, R, H, W2, F, H, G, F, H * F, dH, 2 * F, aux=h, ld_aux=2 * F),
        "up_dgrad": lambda: r("up_dgrad", G, rg, off, 0, H, 2 * F, dH, R, 2 * F, W13, H, 2 * F, G, H, 2 * F * H, dX, H),
        "wgrad_w2": lambda: r("wgrad", G, rg, off, H, F, 0, dY, R, H, act, F, R, 1, F, 0, gW2, F, ogs=H * F),
        "wgrad_w13": lambda: r("wgrad", G, rg, off, 2 * F, H, 0, dH, R, 2 * F, X, H, R, 1, H, 0, gW13, H, ogs=2 * F * H),
    }[a.gemm]


flops = {"gateup": 4 * R * H * F, "down": 2 * R * H * F, "down_dgrad": 2 * R * H * F, "up_dgrad": 4 * R * H * F,
         "wgrad_w2": 2 * R * H * F, "wgrad_w13": 4 * R * H * F}[a.gemm]
try:
    import pynvml
    pynvml.nvmlInit()
    nv = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:
    nv = None

variants = []
for v in a.variants:
    name, spec = v.split("=")
    pol, _, ras = spec.partition(":")
    pw = int(pol, 0)  # a GemmParams::policy word, e.g. 0x800 = no wave sync, 0x100 = no N=128 tail MMA
    variants.append((name, ((pw & 0xF) << 12) | (((pw >> 8) & 0xF) << 24) | (int(ras or 0) << 16)))
results = {n: [] for n, _ in variants}


def run(kind_bits, secs):
    fn = call(kind_bits)
    fn()
    torch.cuda.synchronize()
    t0 = time.time()
    n = 0
    clk, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            if nv is not None:
                clk.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
            stop.wait(0.002)
    th = threading.Thread(target=sample)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th.start()
    s.record()
    while time.time() - t0 < secs:
        for _ in range(5):
            fn()
        n += 5
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / n
    mhz = sum(clk[len(clk) // 5:]) / max(1, len(clk) - len(clk) // 5) if clk else float("nan")
    return ms, mhz


run(variants[0][1], 1.0)  # warm the clock into its loaded state
for rnd in range(a.rounds):
    for name, bits in (variants if rnd % 2 == 0 else variants[::-1]):
        results[name].append(run(bits, a.secs))
for name, _ in variants:
    ms = sorted(m for m, _ in results[name])
    mhz = [c for _, c in results[name]]
    kc = sorted(m * c for m, c in results[name])
    print(f"{a.gemm:10s} {name:12s} ms {ms[len(ms)//2]:.4f} (min {ms[0]:.4f})  MHz {sum(mhz)/len(mhz):6.0f}  "
          f"kcycles {kc[len(kc)//2]:8.1f}  TFLOP/s {flops/ms[len(ms)//2]/1e9:7.1f}")
