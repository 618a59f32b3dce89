"""Shard-restore transport A/B on N GPUs (torchrun; dev/measurement tool).

For the Mixtral (E8, C=2E/N) and fine (E64) layer shapes, times a full expert-
granularity shard restore (every rank receives chunk p of each hosted expert from
every peer p: C x S x 2 bytes per peer) through
  * the copy-engine push transport (cudaMemcpyAsync per chunk + readiness flags),
  * the SM push kernel (FSEP_COMM=sm) at several CTA counts,
  * NCCL (torch.distributed all_to_all_single of the same per-peer bytes),
each as received GB/s per GPU = C*S*2*(N-1) / time, max over ranks.
usage: python -m torch.distributed.run --nproc-per-node N tools/transport_probe.py [out.json]"""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
N = world
shapes = {"mixtral": (8, 2, 4096, 14336), "fine": (64, 8, 2048, 1408)}
out = {}


def maxr(v):
    t = torch.tensor([v], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


for name, (E, K, H, F) in shapes.items():
    C = max(K, min(E, 2 * E // N))
    S = 3 * H * F // N
    rx = C * S * 2 * (N - 1)
    res = {"C": C, "chunk_MB": round(S * 2 / 1e6, 3), "recv_MB_per_gpu": round(rx / 1e6, 1)}
    variants = [(f"copy_engine_{k}lane", {"FSEP_CE_STREAMS": str(k)}) for k in (1, 2, 4)] + \
               [(f"sm_push_{c}cta", {"FSEP_COMM": "sm", "FSEP_PUSH_CTAS": str(c)}) for c in (32, 64, 128)]
    for vname, env in variants:
        for k in ("FSEP_COMM", "FSEP_PUSH_CTAS", "FSEP_CE_STREAMS"):
            os.environ.pop(k, None)
        os.environ.update(env)
        layer = FsepLayer(LayerSpec(E, K, H, F, 256, C, world=N, rank=rank))
        layer.connect_torch_distributed()
        w = torch.zeros(F, H, device="cuda", dtype=torch.bfloat16)
        w2 = torch.zeros(H, F, device="cuda", dtype=torch.bfloat16)
        for e in range(E):
            layer.load_expert(e, w, w, w2)
        torch.cuda.synchronize()
        dist.barrier()
        layer.debug_restore_ms(3)
        ms = maxr(layer.debug_restore_ms(10))
        res[vname] = {"ms": round(ms, 3), "GBps_per_gpu": round(rx / (ms * 1e-3) / 1e9, 1)}
        layer.close()
        torch.cuda.empty_cache()
        dist.barrier()
    for k in ("FSEP_COMM", "FSEP_PUSH_CTAS", "FSEP_CE_STREAMS"):
        os.environ.pop(k, None)
    # NCCL: the same bytes per peer as one all-to-all (own chunk included, as the restore does)
    src = torch.empty(N * C * S, device="cuda", dtype=torch.bfloat16)
    dst = torch.empty_like(src)
    for _ in range(3):
        dist.all_to_all_single(dst, src)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        dist.all_to_all_single(dst, src)
    b.record()
    torch.cuda.synchronize()
    ms = maxr(a.elapsed_time(b) / 10)
    res["nccl_all_to_all"] = {"ms": round(ms, 3), "GBps_per_gpu": round(rx / (ms * 1e-3) / 1e9, 1)}
    del src, dst
    torch.cuda.empty_cache()
    out[name] = res
if rank == 0:
    txt = json.dumps({"n_gpus": N, "nccl": ".".join(map(str, torch.cuda.nccl.version())), **out}, indent=1)
    print(txt)
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(txt)
dist.destroy_process_group()
