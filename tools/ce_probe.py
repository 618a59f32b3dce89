"""Copy-engine peer bandwidth probe (dev tool): pull vs push, streams per peer.

Single process driving N GPUs (torch peer copies = cudaMemcpyPeerAsync on the
copy engines).  Prints GB/s per receiving GPU for each variant.
"""
import sys
import torch

N = torch.cuda.device_count()
MB = int(sys.argv[1]) if len(sys.argv) > 1 else 88
CHUNKS = 4
n = MB * (1 << 20) // 2
for i in range(N):
    for j in range(N):
        if i != j:
            assert torch.cuda.can_device_access_peer(i, j)
src = [[torch.randn(n, device=f"cuda:{d}").bfloat16() for _ in range(CHUNKS)] for d in range(N)]
dst = [[torch.empty(n * N, device=f"cuda:{d}", dtype=torch.bfloat16) for _ in range(CHUNKS)] for d in range(N)]


def run(mode, spp, iters=3):
    streams = {(d, p, k): torch.cuda.Stream(device=d if mode == "pull" else p)
               for d in range(N) for p in range(N) if p != d for k in range(spp)}
    for it in range(iters + 1):
        for d in range(N):
            torch.cuda.synchronize(d)
        t0 = [torch.cuda.Event(enable_timing=True) for _ in range(N)]
        t1 = [torch.cuda.Event(enable_timing=True) for _ in range(N)]
        for d in range(N):
            t0[d].record(torch.cuda.current_stream(d))
        for d in range(N):
            for p in range(N):
                if p == d:
                    continue
                for c in range(CHUNKS):
                    piece = n // spp
                    for k in range(spp):
                        st = streams[(d, p, k)]
                        with torch.cuda.stream(st):
                            dst[d][c][p * n + k * piece: p * n + (k + 1) * piece].copy_(
                                src[p][c][k * piece:(k + 1) * piece], non_blocking=True)
        for d in range(N):
            for p in range(N):
                if p != d:
                    for k in range(spp):
                        torch.cuda.current_stream(d).wait_stream(streams[(d, p, k)])
            t1[d].record(torch.cuda.current_stream(d))
        for d in range(N):
            torch.cuda.synchronize(d)
    ms = max(t0[d].elapsed_time(t1[d]) for d in range(N))
    gb = (N - 1) * CHUNKS * n * 2 / 1e9
    print(f"{mode:5s} streams/peer={spp}: {gb:.2f} GB in per GPU, {ms:.2f} ms -> {gb / ms * 1e3:.0f} GB/s per GPU",
          flush=True)


for mode in ("pull", "push"):
    for spp in (1, 2, 4):
        run(mode, spp)
