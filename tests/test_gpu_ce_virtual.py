"""The shipped multi-GPU data plane on ONE GPU: virtual ranks with MP_FSEP_FLAG_COPY_ENGINE.

Real N>1 mode moves the FSEP-specific traffic with copy engines, not SM kernels
(csrc/runtime/fsep_layer.cu push_restore / push_grads):
  * shard restore (unshard): every rank cudaMemcpyAsync-pushes its
    chunk of each expert into the restored slot of every rank hosting it, each copy
    followed by a cuStreamWriteValue32 readiness flag in the destination's memory;
  * the destination's gate-up GEMM producer polls ready[slot][source]
    (wait_group_ready, ld.acquire.sys + proxy fence, bounded) before its first TMA load
    of that expert, so the restore overlaps router, dispatch and the GEMMs;
  * gradient reduce-scatter (reshard): replica gradient chunks are
    pushed into the owners' staging rows under the dW2 / dX GEMMs, then
    grad_rs_sum_kernel sums them in ascending-device order.
The copy-engine flag makes the emulated ranks run exactly that code (copies between
their arenas on one GPU), so the driver's 1-GPU `pytest -m gpu` checks it against
the oracle: routing bit-exact, numerics within 2e-2 -- at configs[0] (8 ranks), the
fine-grained family, a planner-driven multi-step run, and a Mixtral-shaped N=8, C=2
case (reduced tokens per rank) that must also be BIT-IDENTICAL to the device-kernel
transport (same bytes restored, same ascending-device gradient sums).
"""
import json

import numpy as np
import pytest
import torch

from oracle import layer_oracle as LO
from oracle import planner_port as PP
from paper_2602_11686_b200 import planner as PL
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec
from test_gpu_layer import check_numerics, check_routing, make_problem, oracle, run_gpu
from torch_ref import _rel, layer_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["copy_engine", "sm_push"])
def transport(request, monkeypatch):
    """The push transport under test: copy engines (default) or the SM push kernel
    (FSEP_COMM=sm: push_copies_kernel on a side stream, same readiness flags)."""
    if request.param == "sm_push":
        monkeypatch.setenv("FSEP_COMM", "sm")
        monkeypatch.setenv("FSEP_PUSH_PIECE_KB", "64")  # several pieces per chunk at these sizes
    return request.param


@pytest.mark.parametrize("layout", ["even", "static", "planned"])
def test_tiny_config_8_ranks_copy_engine(layout, transport):
    """configs[0]: E8 top-2, H256, F512, 4096 tokens over 8 ranks, Zipf(1.2), copy-engine transport."""
    N, E, K, H, F, T, C = 8, 8, 2, 256, 512, 512, 2
    pb = make_problem(N, E, K, H, F, T, 1.2, seed=42)
    if layout == "even":
        A = PL.even_replication_layout(N, E, C)
    elif layout == "static":
        A = PL.static_ep_layout(N, E, C)
    else:
        A = PL.plan_layout(oracle(pb, K, PL.even_replication_layout(N, E, C), C)["routing"].R, C)
    ref = oracle(pb, K, A, C)
    layer, y, dx = run_gpu(pb, N, E, K, H, F, T, C, A, copy_engine=True)
    assert layer.check() == 0
    check_routing(layer, ref, N, T, K, C)
    check_numerics(layer, ref, y, dx, N, T, H, E)
    # the restored experts are exactly the unsharded weights of the hosted experts
    flat = 3 * H * F
    for d in range(N):
        rest = layer.read("restored", d).view(np.uint16).reshape(C, flat)
        hosted = [e for e in range(E) if A[e, d]]
        for c, e in enumerate(hosted):
            w1 = pb["w1"][e].view(torch.int16).numpy().astype(np.uint16)
            w13 = rest[c, :2 * F * H].reshape(F // 128, 2, 128, H)
            assert np.array_equal(w13[:, 0].reshape(F, H), w1), (d, c, e)
    layer.close()


def test_fine_grained_topk8_copy_engine(transport):
    """E64 top-8 family (token de-duplication on), 4 ranks, C=16, planned layout."""
    N, E, K, H, F, T, C = 4, 64, 8, 256, 384, 256, 16
    pb = make_problem(N, E, K, H, F, T, 1.2, seed=5)
    A = PL.plan_layout(oracle(pb, K, PL.even_replication_layout(N, E, C), C)["routing"].R, C)
    ref = oracle(pb, K, A, C)
    layer, y, dx = run_gpu(pb, N, E, K, H, F, T, C, A, copy_engine=True)
    assert layer.check() == 0
    check_routing(layer, ref, N, T, K, C)
    check_numerics(layer, ref, y, dx, N, T, H, E)
    layer.close()


def test_planner_steps_copy_engine(transport):
    """Attached planner, 3 steps, layout changes every step: each restore epoch's
    readiness flags gate the GEMMs of that step only; every step vs the oracle."""
    N, E, K, H, F, T, C = 4, 8, 2, 256, 256, 256, 3
    spec = LayerSpec(E, K, H, F, T, C, world=N, virtual=True, copy_engine=True)
    layer = FsepLayer(spec)
    pb = make_problem(N, E, K, H, F, T, 1.5, seed=9)
    for e in range(E):
        layer.load_expert(e, pb["w1"][e].cuda().contiguous(), pb["w3"][e].cuda().contiguous(),
                          pb["w2"][e].cuda().contiguous())
    layer.load_router(pb["wg"].cuda())
    cfg = PL.Config(json.dumps({"topology": {"n_nodes": 1, "devices_per_node": N, "b_intra": 9e11, "b_inter": 9e11},
                                "cost": {"v_comm": 2 * H, "v_comp": 6 * H * F, "b_comp": 1.6354e15},
                                "model": {"n_experts": E, "capacity": C}, "planner": {"seed": 7}}))
    layer.attach_planner(cfg, layer=0)
    x = torch.cat(pb["xs"]).cuda()
    dy = torch.cat(pb["dys"]).cuda()
    y, dx = torch.empty_like(x), torch.empty_like(x)
    topo = PP.Topology(1, N, 9e11, 9e11)
    params = PP.CostParams(2 * H, 6 * H * F, 1.6354e15)
    history, layouts = [], []
    A = np.array(PP.even_replication_layout(topo, E, C), dtype=np.uint8)
    for step in range(3):
        rng = np.random.default_rng(200 + step)
        biases = [LO.make_bias(rng, T, E, 1.5, rng.permutation(E)) for _ in range(N)]
        layer.forward(x, torch.from_numpy(np.concatenate(biases)).cuda(), T, y)
        layer.backward(dy, dx)
        torch.cuda.synchronize()
        assert layer.check() == 0
        assert np.array_equal(layer.read("layout", 0).reshape(E, N), A), step
        layouts.append(A.copy())
        pbs = dict(pb, biases=biases)
        ref = oracle(pbs, K, A, C)
        check_routing(layer, ref, N, T, K, C)
        check_numerics(layer, ref, y, dx, N, T, H, E)
        history.append(layer.histogram().astype(np.int64).tolist())
        A = np.array(PP.plan_layout(history, topo, params, C, PP.SearchSpec(2, PP.mix_seed(7, 0x6C617972, 0))),
                     dtype=np.uint8)
    assert any(not np.array_equal(layouts[0], a) for a in layouts[1:]), "the planner never changed the layout"
    layer.close()


def test_soak_200_steps_drifting_copy_engine(transport):
    """200 steps with the planner attached and the routing skew re-drawn every step:
    200 restore epochs of readiness flags and reduce-scatter pushes.  Every step: no
    device-detected failure and the layout the host planner predicts; steps 0, 99 and
    199 in full vs the oracle."""
    N, E, K, H, F, T, C = 4, 8, 2, 256, 256, 128, 3
    layer = FsepLayer(LayerSpec(E, K, H, F, T, C, world=N, virtual=True, copy_engine=True))
    pb = make_problem(N, E, K, H, F, T, 1.2, seed=21)
    for e in range(E):
        layer.load_expert(e, pb["w1"][e].cuda().contiguous(), pb["w3"][e].cuda().contiguous(),
                          pb["w2"][e].cuda().contiguous())
    layer.load_router(pb["wg"].cuda())
    cfg = PL.Config(json.dumps({"topology": {"n_nodes": 1, "devices_per_node": N, "b_intra": 9e11, "b_inter": 9e11},
                                "cost": {"v_comm": 2 * H, "v_comp": 6 * H * F, "b_comp": 1.6354e15},
                                "model": {"n_experts": E, "capacity": C}, "planner": {"seed": 3}}))
    layer.attach_planner(cfg, layer=0)
    x = torch.cat(pb["xs"]).cuda()
    dy = torch.cat(pb["dys"]).cuda()
    y, dx = torch.empty_like(x), torch.empty_like(x)
    topo = PP.Topology(1, N, 9e11, 9e11)
    params = PP.CostParams(2 * H, 6 * H * F, 1.6354e15)
    history, changes = [], 0
    A = np.array(PP.even_replication_layout(topo, E, C), dtype=np.uint8)
    for step in range(200):
        rng = np.random.default_rng(1000 + step)
        biases = [LO.make_bias(rng, T, E, 0.6 + 0.9 * rng.random(), rng.permutation(E)) for _ in range(N)]
        layer.forward(x, torch.from_numpy(np.concatenate(biases)).cuda(), T, y)
        layer.backward(dy, dx)
        assert layer.check() == 0, step
        assert np.array_equal(layer.read("layout", 0).reshape(E, N), A), step
        if step in (0, 99, 199):
            ref = oracle(dict(pb, biases=biases), K, A, C)
            check_routing(layer, ref, N, T, K, C)
            check_numerics(layer, ref, y, dx, N, T, H, E)
        history.append(layer.histogram().astype(np.int64).tolist())
        nxt = np.array(PP.plan_layout(history, topo, params, C, PP.SearchSpec(2, PP.mix_seed(3, 0x6C617972, 0))),
                       dtype=np.uint8)
        changes += int(not np.array_equal(nxt, A))
        A = nxt
    assert changes >= 10, f"the planner changed the layout only {changes} times"
    layer.close()


def _mixtral_n8_run(copy_engine, w, xs, dys, biases, A, E, K, H, F, T, C, N):
    layer = FsepLayer(LayerSpec(E, K, H, F, T, C, world=N, virtual=True, copy_engine=copy_engine))
    for e in range(E):
        layer.load_expert(e, *w(e))
    layer.load_router(w("g"))
    layer.set_layout(A)
    x = torch.cat(xs)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    layer.forward(x, torch.from_numpy(np.concatenate(biases)).cuda(), T, y)
    layer.backward(torch.cat(dys), dx)
    torch.cuda.synchronize()
    assert layer.check() == 0
    out = {"y": y, "dx": dx, "grads": [layer.expert_grad(e) for e in range(E)],
           "dwg": [layer.router_grad(v) for v in range(N)],
           "idx": [layer.read("topk_idx", v).view(np.int32).reshape(T, K) for v in range(N)],
           "slot": [layer.read("slot_dst", v).view(np.uint32).reshape(T, K) for v in range(N)]}
    torch.cuda.synchronize()
    layer.close()
    torch.cuda.empty_cache()
    return out


def test_mixtral_shape_8_ranks_c2_copy_engine(transport):
    """Mixtral expert shape (H4096, F14336, E8 top-2), N=8, C=2, 512 tokens per rank:
    copy-engine transport == device-kernel transport bit for bit, and both within 2e-2
    of the torch fp32 reference on the oracle's routing (every output and gradient)."""
    N, E, K, H, F, T, C = 8, 8, 2, 4096, 14336, 512, 2
    g = torch.Generator(device="cuda").manual_seed(3)
    W = {e: ((torch.randn(F, H, device="cuda", generator=g) / H ** 0.5).bfloat16(),
             (torch.randn(F, H, device="cuda", generator=g) / H ** 0.5).bfloat16(),
             (torch.randn(H, F, device="cuda", generator=g) / F ** 0.5).bfloat16()) for e in range(E)}
    W["g"] = (torch.randn(E, H, device="cuda", generator=g) * 0.02).bfloat16()
    xs = [torch.randn(T, H, device="cuda", generator=g).bfloat16() for _ in range(N)]
    dys = [(torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16() for _ in range(N)]
    rng = np.random.default_rng(17)
    perm = rng.permutation(E)
    biases = [LO.make_bias(rng, T, E, 1.2, perm) for _ in range(N)]
    # routing from the oracle (bit-exact), layout planned from it (skewed -> replicated hot experts)
    idx_l, w_l = [], []
    for v in range(N):
        lg = LO.router_logits(xs[v].float().cpu().numpy(), W["g"].float().cpu().numpy(), biases[v])
        i_, w_ = LO.topk(lg, K)
        idx_l.append(i_)
        w_l.append(w_)
    rt0 = LO.route(idx_l, w_l, PL.even_replication_layout(N, E, C), E, C)
    A = PL.plan_layout(rt0.R, C)
    rt = LO.route(idx_l, w_l, A, E, C)
    ce = _mixtral_n8_run(True, W.get, xs, dys, biases, A, E, K, H, F, T, C, N)
    for v in range(N):
        assert np.array_equal(ce["idx"][v], idx_l[v])
        assert np.array_equal(ce["slot"][v] >> 24, rt.slot_dev[v])
        assert np.array_equal(ce["slot"][v] & 0xFFFFFF, rt.slot_row[v])
    import os
    os.environ.pop("FSEP_COMM", None)  # the reference run: device-kernel transport
    kern = _mixtral_n8_run(False, W.get, xs, dys, biases, A, E, K, H, F, T, C, N)
    assert torch.equal(ce["y"], kern["y"]) and torch.equal(ce["dx"], kern["dx"])
    for e in range(E):
        for a, b in zip(ce["grads"][e], kern["grads"][e]):
            assert torch.equal(a, b), f"expert {e} gradient differs between transports"
    for v in range(N):
        assert torch.equal(ce["dwg"][v], kern["dwg"][v])
    errs = {}

    def on_expert(e, dW1, dW3, dW2):
        for n, a, b in zip(("dW1", "dW3", "dW2"), ce["grads"][e], (dW1, dW3, dW2)):
            errs[f"{n}[{e}]"] = _rel(a, b)

    ys, dxs, dWgs = layer_ref(xs, dys, W["g"], W.get, [torch.from_numpy(i).long().cuda() for i in idx_l],
                              [torch.from_numpy(w_).cuda() for w_ in w_l], on_expert=on_expert)
    for v in range(N):
        errs[f"y{v}"] = _rel(ce["y"][v * T:(v + 1) * T], ys[v])
        errs[f"dx{v}"] = _rel(ce["dx"][v * T:(v + 1) * T], dxs[v])
        errs[f"dWg{v}"] = _rel(ce["dwg"][v], dWgs[v])
    worst = max(errs, key=errs.get)
    assert errs[worst] < 2e-2, f"{worst}: {errs[worst]:.3e}"
