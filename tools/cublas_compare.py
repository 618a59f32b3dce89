"""cuBLAS reference for the six expert GEMMs of one layer step (dev tool).

Times torch.matmul (cuBLAS, bf16 in / fp32 accumulate) per expert for the same
shapes tools/gemm_perf.py runs through our grouped tcgen05 kernel, so the two
can be compared on one box:  python tools/cublas_compare.py H F G rows
(wgrad outputs are bf16 here -- cuBLAS would need a separate fp32-output path --
so cuBLAS does slightly less output work than our fp32-gradient wgrad).
"""
import sys

import torch

H, F, G, rows = (int(v) for v in sys.argv[1:5])
dev = "cuda"
X = [torch.randn(rows, H, device=dev).bfloat16() for _ in range(G)]
W13 = [(torch.randn(2 * F, H, device=dev) / H ** 0.5).bfloat16() for _ in range(G)]
W2 = [(torch.randn(H, F, device=dev) / F ** 0.5).bfloat16() for _ in range(G)]
act = [torch.randn(rows, F, device=dev).bfloat16() for _ in range(G)]
dY = [torch.randn(rows, H, device=dev).bfloat16() for _ in range(G)]
dH = [torch.randn(rows, 2 * F, device=dev).bfloat16() for _ in range(G)]

tests = {
    "gateup": (lambda: [X[g] @ W13[g].t() for g in range(G)], 2 * rows * G * H * 2 * F),
    "down": (lambda: [act[g] @ W2[g].t() for g in range(G)], 2 * rows * G * H * F),
    "down_dgrad": (lambda: [dY[g] @ W2[g] for g in range(G)], 2 * rows * G * H * F),
    "up_dgrad": (lambda: [dH[g] @ W13[g] for g in range(G)], 2 * rows * G * H * 2 * F),
    "wgrad_w2": (lambda: [dY[g].t() @ act[g] for g in range(G)], 2 * rows * G * H * F),
    "wgrad_w13": (lambda: [dH[g].t() @ X[g] for g in range(G)], 2 * rows * G * H * 2 * F),
}


def bench(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


tot_ms = tot_fl = 0.0
for name, (fn, fl) in tests.items():
    ms = bench(fn)
    tot_ms += ms
    tot_fl += fl
    print(f"cublas {name:12s} {ms:8.3f} ms  {fl / ms / 1e9:8.1f} TFLOP/s")
print(f"cublas total {tot_ms:.3f} ms {tot_fl / tot_ms / 1e9:.1f} TFLOP/s")
