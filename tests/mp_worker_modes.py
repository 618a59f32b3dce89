"""Worker for tests/test_gpu_multiprocess.py::test_real_multi_gpu_modes (torchrun,
one process per GPU, copy-engine communication).  Checks, in real multi-GPU mode:

* layer chaining (mp_fsep_layer_chain, PAPER Fig.5): a 2-layer step with layer 2's
  restore issued after layer 1's gate-up GEMM gives bit-identical outputs and
  gradients to the unchained step;
* pure-EP resident experts (MP_FSEP_FLAG_RESIDENT_EXPERTS): y / dx match the CPU
  oracle on the static layout, and a second step (no restore) reproduces the
  first bit for bit;
* local-first routing (MP_FSEP_FLAG_LOCAL_FIRST): every slot's destination matches
  the oracle's local-first variant bit for bit;
* deferred gradient reduce-scatter (MP_FSEP_FLAG_DEFER_RS, PAPER Fig.5(e)): layer 2's
  reduce-scatter completed under layer 1's backward gives bit-identical gradients;
* the SM push transport (FSEP_COMM=sm) and the NCCL transport (FSEP_COMM=nccl:
  grouped ncclSend/ncclRecv restore and gradient exchange) are bit-identical to the
  copy engines;
* a 100-step soak with the planner attached and the routing skew re-drawn every step
  (healthy every 10th step; the last step vs the oracle on the layout it used);
* no device-detected failure (barrier / readiness timeouts, overflow, memory guards).
Exits non-zero on the first mismatch."""
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

E, K, H, F, T = 8, 2, 256, 256, 256


def weights(seed):
    g = torch.Generator().manual_seed(seed)
    wg = (torch.randn(E, H, generator=g) * 0.02).bfloat16()
    w1 = (torch.randn(E, F, H, generator=g) / H ** 0.5).bfloat16()
    w3 = (torch.randn(E, F, H, generator=g) / H ** 0.5).bfloat16()
    w2 = (torch.randn(E, H, F, generator=g) / F ** 0.5).bfloat16()
    return wg, w1, w3, w2


def make_layer(world, rank, C, W, **kw):
    layer = FsepLayer(LayerSpec(E, K, H, F, T, C, world=world, rank=rank, virtual=False, **kw))
    layer.connect_torch_distributed()
    wg, w1, w3, w2 = W
    for e in range(E):
        layer.load_expert(e, w1[e].cuda().contiguous(), w3[e].cuda().contiguous(), w2[e].cuda().contiguous())
    layer.load_router(wg.cuda())
    return layer


def config(world, C):
    return PL.Config(json.dumps({"topology": {"n_nodes": 1, "devices_per_node": world, "b_intra": 9e11,
                                              "b_inter": 9e11},
                                 "cost": {"v_comm": 2 * H, "v_comp": 6 * H * F, "b_comp": 1.6354e15},
                                 "model": {"n_experts": E, "capacity": C}, "planner": {"seed": 7}}))


def inputs(rank, step):
    gx = torch.Generator().manual_seed(1000 * step + rank)
    x = torch.randn(T, H, generator=gx).bfloat16()
    dy = (torch.randn(T, H, generator=gx) * 0.1).bfloat16()
    rng = np.random.default_rng(1000 * step + rank)
    bias = LO.make_bias(rng, T, E, 1.2, np.random.default_rng(5).permutation(E))
    return x, dy, bias


def two_layer_steps(world, rank, chain, defer_rs=False):
    C = 4
    layers = [make_layer(world, rank, C, weights(11 + l), defer_rs=defer_rs) for l in range(2)]
    for l, layer in enumerate(layers):
        layer.attach_planner(config(world, C), layer=l)
    if chain:
        layers[0].chain(layers[1])
    outs = []
    for step in range(3):
        x, dy, bias = inputs(rank, step)
        x_d, dy_d, b_d = x.cuda(), dy.cuda(), torch.from_numpy(bias).cuda()
        y1 = torch.empty_like(x_d)
        y2 = torch.empty_like(x_d)
        dx2 = torch.empty_like(x_d)
        dx1 = torch.empty_like(x_d)
        layers[0].forward(x_d, b_d, T, y1)
        layers[1].forward(y1, b_d, T, y2)
        layers[1].backward(dy_d, dx2)
        layers[0].backward(dx2, dx1)
        torch.cuda.synchronize()
        grads = [torch.stack(t).cpu() for t in zip(*[layers[1].expert_grad(e) for e in range(E)])]
        outs.append((y2.cpu(), dx1.cpu(), grads))
    for layer in layers:
        assert layer.check() == 0
        layer.close()
    return outs


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))

    # 1. chaining is bit-identical to the unchained schedule
    a = two_layer_steps(world, rank, chain=False)
    b = two_layer_steps(world, rank, chain=True)
    c = two_layer_steps(world, rank, chain=True, defer_rs=True)
    os.environ["FSEP_COMM"] = "sm"
    d = two_layer_steps(world, rank, chain=True)
    os.environ["FSEP_COMM"] = "nccl"
    n = two_layer_steps(world, rank, chain=True)
    del os.environ["FSEP_COMM"]
    for tag, other in (("chained", b), ("deferred reduce-scatter", c), ("SM push transport", d),
                       ("NCCL transport", n)):
        for step, (u, v) in enumerate(zip(a, other)):
            assert torch.equal(u[0], v[0]) and torch.equal(u[1], v[1]), f"{tag} outputs differ (step {step})"
            for gu, gv in zip(u[2], v[2]):
                assert torch.equal(gu, gv), f"{tag} gradients differ (step {step})"

    # 2. pure EP: resident experts, no restore after the first step, no reduce-scatter
    C = E // world
    W = weights(23)
    layer = make_layer(world, rank, C, W, resident=True)
    A = PL.static_ep_layout(world, E, C)
    layer.set_layout(A)
    x, dy, bias = inputs(rank, 0)
    x_d, dy_d, b_d = x.cuda(), dy.cuda(), torch.from_numpy(bias).cuda()
    res = []
    for _ in range(2):
        y = torch.empty_like(x_d)
        dx = torch.empty_like(x_d)
        layer.forward(x_d, b_d, T, y)
        layer.backward(dy_d, dx)
        torch.cuda.synchronize()
        res.append((y.cpu(), dx.cpu()))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1]), "resident step 2 differs"
    allx = [None] * world
    dist.all_gather_object(allx, (x.float().numpy(), dy.float().numpy(), bias))
    wg, w1, w3, w2 = (t.float().numpy() for t in W)
    ref = LO.layer_step([v[0] for v in allx], [v[2] for v in allx], wg, w1, w3, w2, K, A, C, [v[1] for v in allx])
    for name, got, want in (("y", res[0][0], ref["y"][rank]), ("dx", res[0][1], ref["dx"][rank])):
        err = float(np.abs(got.float().numpy() - want).max() / max(np.abs(want).max(), 1e-30))
        assert err < 2e-2, f"pure EP {name} rel err {err}"
    layer.close()

    # 3. local-first routing: slot destinations match the oracle variant
    C = 4
    layer = make_layer(world, rank, C, weights(31), local_first=True)
    A = PL.even_replication_layout(world, E, C)
    layer.set_layout(A)
    y = torch.empty_like(x_d)
    dx = torch.empty_like(x_d)
    layer.forward(x_d, b_d, T, y)
    layer.backward(dy_d, dx)
    torch.cuda.synchronize()
    W = weights(31)
    wg, w1, w3, w2 = (t.float().numpy() for t in W)
    ref = LO.layer_step([v[0] for v in allx], [v[2] for v in allx], wg, w1, w3, w2, K, A, C, [v[1] for v in allx],
                        local_first=True)
    code = layer.read("slot_dst").view(np.uint32).reshape(T, K)
    assert np.array_equal(code >> 24, ref["routing"].slot_dev[rank]), "local-first slot devices differ"
    assert np.array_equal(code & 0xFFFFFF, ref["routing"].slot_row[rank]), "local-first slot rows differ"
    err = float(np.abs(y.cpu().float().numpy() - ref["y"][rank]).max() / np.abs(ref["y"][rank]).max())
    assert err < 2e-2, f"local-first y rel err {err}"
    layer.close()

    # 4. soak: 100 steps, planner attached, routing skew re-drawn every step -- every 10th
    # step healthy, and the last step vs the oracle on the layout the layer used
    C = E // world + 1  # one spare slot per device: the planner has replicas to move
    W = weights(41)
    layer = make_layer(world, rank, C, W)
    layer.attach_planner(config(world, C), layer=0)
    y = torch.empty_like(x_d)
    dx = torch.empty_like(x_d)
    for step in range(100):
        rng = np.random.default_rng(7000 + 31 * step + rank)
        bias = LO.make_bias(rng, T, E, 0.6 + 0.9 * np.random.default_rng(step).random(),
                            np.random.default_rng(step).permutation(E))
        layer.forward(x_d, torch.from_numpy(bias).cuda(), T, y)
        layer.backward(dy_d, dx)
        if step % 10 == 9:
            assert layer.check() == 0, f"soak step {step}: device-detected failure"
    torch.cuda.synchronize()
    A = layer.read("layout").reshape(E, world)
    allb = [None] * world
    dist.all_gather_object(allb, bias)
    wg, w1, w3, w2 = (t.float().numpy() for t in W)
    ref = LO.layer_step([v[0] for v in allx], allb, wg, w1, w3, w2, K, A, C, [v[1] for v in allx])
    for name, got, want in (("y", y, ref["y"][rank]), ("dx", dx, ref["dx"][rank])):
        err = float(np.abs(got.cpu().float().numpy() - want).max() / max(np.abs(want).max(), 1e-30))
        assert err < 2e-2, f"soak {name} rel err {err}"
    layer.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("modes ok", flush=True)


if __name__ == "__main__":
    main()
