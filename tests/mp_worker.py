"""Worker for tests/test_gpu_multiprocess.py: one process per GPU (torchrun),
real-mode FSEP layer (CUDA IPC peer memory + barrier kernels).  Every rank runs
two steps with the attached planner, then dumps its routing arrays, outputs and
gradient shards for the parent test to compare against the CPU oracle."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import layer_oracle as LO  # noqa: E402
from paper_2602_11686_b200 import planner as PL  # noqa: E402
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec  # noqa: E402


def main():
    out_dir = Path(sys.argv[1])
    E, K, H, F, T, C = (int(v) for v in sys.argv[2:8])
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    g = torch.Generator().manual_seed(11)
    wg = (torch.randn(E, H, generator=g) * 0.02).bfloat16()
    w1 = (torch.randn(E, F, H, generator=g) / H ** 0.5).bfloat16()
    w3 = (torch.randn(E, F, H, generator=g) / H ** 0.5).bfloat16()
    w2 = (torch.randn(E, H, F, generator=g) / F ** 0.5).bfloat16()
    layer = FsepLayer(LayerSpec(E, K, H, F, T, C, world=world, rank=rank, virtual=False))
    layer.connect_torch_distributed()
    for e in range(E):
        layer.load_expert(e, w1[e].cuda().contiguous(), w3[e].cuda().contiguous(), w2[e].cuda().contiguous())
    layer.load_router(wg.cuda())
    cfg = PL.Config(json.dumps({"topology": {"n_nodes": 1, "devices_per_node": world, "b_intra": 9e11,
                                             "b_inter": 9e11},
                                "cost": {"v_comm": 2 * H, "v_comp": 6 * H * F, "b_comp": 1.6354e15},
                                "model": {"n_experts": E, "capacity": C}, "planner": {"seed": 7}}))
    layer.attach_planner(cfg, layer=0)
    for step in range(2):
        gx = torch.Generator().manual_seed(1000 * step + rank)
        x = torch.randn(T, H, generator=gx).bfloat16()
        dy = (torch.randn(T, H, generator=gx) * 0.1).bfloat16()
        rng = np.random.default_rng(1000 * step + rank)
        bias = LO.make_bias(rng, T, E, 1.2, np.random.default_rng(5).permutation(E))
        y = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
        dx = torch.empty_like(y)
        x_d, b_d, dy_d = x.cuda(), torch.from_numpy(bias).cuda(), dy.cuda()  # x must live until backward
        layer.forward(x_d, b_d, T, y)
        layer.backward(dy_d, dx)
        torch.cuda.synchronize()
        dw = [torch.stack(t) for t in zip(*[layer.expert_grad(e) for e in range(E)])]
        torch.cuda.synchronize()
        for t in dw:  # each rank contributes its shard chunk; the sum is the full gradient
            dist.all_reduce(t)
        np.savez(out_dir / f"r{rank}_s{step}.npz", x=x.float().numpy(), dy=dy.float().numpy(), bias=bias,
                 y=y.float().cpu().numpy(), dx=dx.float().cpu().numpy(),
                 idx=layer.read("topk_idx").view(np.int32).reshape(T, K),
                 slot=layer.read("slot_dst").view(np.uint32).reshape(T, K),
                 seg_rows=layer.read("seg_rows").view(np.int32), layout=layer.read("layout").reshape(E, world),
                 R=layer.histogram(), dwg=layer.router_grad().cpu().numpy(),
                 dw1=dw[0].cpu().numpy(), dw3=dw[1].cpu().numpy(), dw2=dw[2].cpu().numpy(),
                 barrier=layer.read("barrier_status").view(np.uint32))
    assert layer.check() == 0  # no barrier / readiness timeout, no receive overflow
    if rank == 0:
        np.savez(out_dir / "weights.npz", wg=wg.float().numpy(), w1=w1.float().numpy(), w3=w3.float().numpy(),
                 w2=w2.float().numpy())
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
