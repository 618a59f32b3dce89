"""FSEP layer step on the GPU (through the C ABI) vs the CPU oracle.

Bit-exact: top-k expert ids, R (histograms), every token-slot's destination
(device, row), the per-device segment layout, the planner's layouts.
Tolerance (bf16 storage, fp32 accumulation): max|gpu - oracle| / max|oracle|
<= 2e-2 for y, dx, expert and router gradients (SURVEY/north star: 2e-2)."""
import json

import numpy as np
import pytest
import torch

from oracle import layer_oracle as LO
from oracle import planner_port as PP
from paper_2602_11686_b200 import planner as PL
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec

pytestmark = pytest.mark.gpu
TOL = 2e-2


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def make_problem(N, E, K, H, F, T, alpha, seed):
    g = torch.Generator().manual_seed(seed)
    wg = (torch.randn(E, H, generator=g) * 0.02).bfloat16()
    w1 = (torch.randn(E, F, H, generator=g) / H ** 0.5).bfloat16()
    w3 = (torch.randn(E, F, H, generator=g) / H ** 0.5).bfloat16()
    w2 = (torch.randn(E, H, F, generator=g) / F ** 0.5).bfloat16()
    xs = [(torch.randn(T, H, generator=g)).bfloat16() for _ in range(N)]
    dys = [(torch.randn(T, H, generator=g) * 0.1).bfloat16() for _ in range(N)]
    rng = np.random.default_rng(seed)
    perm = rng.permutation(E)
    biases = [LO.make_bias(rng, T, E, alpha, perm) for _ in range(N)]
    return dict(wg=wg, w1=w1, w3=w3, w2=w2, xs=xs, dys=dys, biases=biases)


def run_gpu(pb, N, E, K, H, F, T, C, A, virtual=True, resident=False, local_first=False, copy_engine=False):
    spec = LayerSpec(E, K, H, F, T, C, world=N, virtual=virtual, resident=resident, local_first=local_first,
                     copy_engine=copy_engine)
    layer = FsepLayer(spec)
    for e in range(E):
        layer.load_expert(e, pb["w1"][e].cuda().contiguous(), pb["w3"][e].cuda().contiguous(),
                          pb["w2"][e].cuda().contiguous())
    layer.load_router(pb["wg"].cuda())
    layer.set_layout(A)
    x = torch.cat(pb["xs"]).cuda()
    bias = torch.from_numpy(np.concatenate(pb["biases"])).cuda()
    dy = torch.cat(pb["dys"]).cuda()
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    layer.forward(x, bias, T, y)
    layer.backward(dy, dx)
    torch.cuda.synchronize()
    return layer, y, dx


def oracle(pb, K, A, C, local_first=False):
    f32 = lambda t: t.float().numpy()
    return LO.layer_step([f32(x) for x in pb["xs"]], pb["biases"], f32(pb["wg"]), f32(pb["w1"]), f32(pb["w3"]),
                         f32(pb["w2"]), K, A, C, [f32(d) for d in pb["dys"]], local_first=local_first)


def check_routing(layer, ref, N, T, K, C):
    rt = ref["routing"]
    for v in range(N):
        idx = layer.read("topk_idx", v).view(np.int32).reshape(T, K)
        assert np.array_equal(idx, rt.idx[v]), f"top-k ids differ on rank {v}"
        code = layer.read("slot_dst", v).view(np.uint32).reshape(T, K)
        assert np.array_equal(code >> 24, rt.slot_dev[v]), f"slot devices differ on rank {v}"
        assert np.array_equal(code & 0xFFFFFF, rt.slot_row[v]), f"slot rows differ on rank {v}"
        assert np.array_equal(layer.read("seg_rows", v).view(np.int32), rt.seg_rows[v])
        assert np.array_equal(layer.read("seg_off", v).view(np.int32), rt.seg_off[v])
        assert np.array_equal(layer.read("slot_expert", v).view(np.int32), rt.slot_expert[v])
        assert layer.read("status", v).view(np.int32)[0] == 0
    # every receive row knows its origin slot (drives the GEMM epilogue's return scatter);
    # padding rows are marked -1
    for d in range(N):
        src = layer.read("row_src", d).view(np.int32)
        seg_rows = rt.seg_rows[d]
        seg_off = rt.seg_off[d]
        for c in range(len(seg_rows)):
            pad_end = seg_off[c] + (seg_rows[c] + 127) // 128 * 128
            assert (src[seg_off[c] + seg_rows[c]:pad_end] == -1).all(), f"pad rows of slot {c} on rank {d}"
    for v in range(N):
        want = (v << 26) | np.arange(T * K, dtype=np.int64).reshape(T, K)
        for d in range(N):
            src = layer.read("row_src", d).view(np.int32)
            m = rt.slot_dev[v] == d
            assert np.array_equal(src[rt.slot_row[v][m]], want[m]), f"row origins of rank {v} on rank {d}"
    assert np.array_equal(layer.histogram(), rt.R)


def check_numerics(layer, ref, y, dx, N, T, H, E):
    yg = y.float().cpu().numpy().reshape(N, T, H)
    dxg = dx.float().cpu().numpy().reshape(N, T, H)
    for v in range(N):
        assert rel(yg[v], ref["y"][v]) < TOL
        assert rel(dxg[v], ref["dx"][v]) < TOL
        assert rel(layer.router_grad(v).cpu().numpy(), ref["dWg"][v]) < TOL
    for e in range(E):
        dw1, dw3, dw2 = (t.cpu().numpy() for t in layer.expert_grad(e))
        torch.cuda.synchronize()
        assert rel(dw1, ref["dW1"][e]) < TOL, e
        assert rel(dw3, ref["dW3"][e]) < TOL, e
        assert rel(dw2, ref["dW2"][e]) < TOL, e


@pytest.mark.parametrize("layout", ["even", "static", "planned"])
def test_tiny_config_8_virtual_ranks(layout):
    """configs[0]: 8 experts top-2, H 256, F 512, 4096 tokens over 8 simulated devices, Zipf(1.2)."""
    N, E, K, H, F, T, C = 8, 8, 2, 256, 512, 512, 2
    pb = make_problem(N, E, K, H, F, T, 1.2, seed=42)
    if layout == "even":
        A = PL.even_replication_layout(N, E, C)
    elif layout == "static":
        A = PL.static_ep_layout(N, E, C)
    else:  # plan from this step's own histogram (as the next step would)
        ref0 = oracle(pb, K, PL.even_replication_layout(N, E, C), C)
        A = PL.plan_layout(ref0["routing"].R, C)
    ref = oracle(pb, K, A, C)
    layer, y, dx = run_gpu(pb, N, E, K, H, F, T, C, A)
    check_routing(layer, ref, N, T, K, C)
    check_numerics(layer, ref, y, dx, N, T, H, E)
    layer.close()


def test_single_device_all_experts():
    N, E, K, H, F, T, C = 1, 8, 2, 512, 256, 1000, 8  # ragged T (not a multiple of 128)
    pb = make_problem(N, E, K, H, F, T, 1.2, seed=3)
    A = PL.even_replication_layout(N, E, C)
    ref = oracle(pb, K, A, C)
    layer, y, dx = run_gpu(pb, N, E, K, H, F, T, C, A)
    check_routing(layer, ref, N, T, K, C)
    check_numerics(layer, ref, y, dx, N, T, H, E)
    layer.close()


def test_fine_grained_topk8():
    """Fine-grained shape family (E=64, K=8) at reduced H/F, 4 virtual ranks, C=16."""
    N, E, K, H, F, T, C = 4, 64, 8, 256, 384, 256, 16
    pb = make_problem(N, E, K, H, F, T, 1.2, seed=5)
    A = PL.plan_layout(oracle(pb, K, PL.even_replication_layout(N, E, C), C)["routing"].R, C)
    ref = oracle(pb, K, A, C)
    layer, y, dx = run_gpu(pb, N, E, K, H, F, T, C, A)
    check_routing(layer, ref, N, T, K, C)
    check_numerics(layer, ref, y, dx, N, T, H, E)
    layer.close()


def test_planner_lag_on_device():
    """Attached planner: step t+1 runs on plan_layout(R_t) (sim.cpp:114-131)."""
    N, E, K, H, F, T, C = 4, 8, 2, 256, 256, 256, 4
    spec = LayerSpec(E, K, H, F, T, C, world=N, virtual=True)
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
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    dy = torch.cat(pb["dys"]).cuda()
    topo = PP.Topology(1, N, 9e11, 9e11)
    params = PP.CostParams(2 * H, 6 * H * F, 1.6354e15)
    history = []
    expected = np.array(PP.even_replication_layout(topo, E, C), dtype=np.uint8)
    for step in range(3):
        rng = np.random.default_rng(100 + step)
        bias = torch.from_numpy(np.concatenate([LO.make_bias(rng, T, E, 1.5, rng.permutation(E)) for _ in range(N)]))
        layer.forward(x, bias.cuda(), T, y)
        layer.backward(dy, dx)
        torch.cuda.synchronize()
        assert np.array_equal(layer.read("layout", 0).reshape(E, N), expected), step
        R = layer.histogram()
        history.append(R.astype(np.int64).tolist())
        spec_ = PP.SearchSpec(2, PP.mix_seed(7, 0x6C617972, 0))
        expected = np.array(PP.plan_layout(history, topo, params, C, spec_), dtype=np.uint8)
    layer.close()


def test_pure_ep_resident_experts():
    """Pure-EP baseline mode (E == N*C, one host per expert, experts stay restored,
    no gradient reduce-scatter): same numerics as FSEP; a second step reuses the
    resident experts and must reproduce the first step exactly."""
    N, E, K, H, F, T, C = 4, 8, 2, 256, 256, 384, 2
    pb = make_problem(N, E, K, H, F, T, 1.2, seed=13)
    A = PL.static_ep_layout(N, E, C)
    ref = oracle(pb, K, A, C)
    layer, y, dx = run_gpu(pb, N, E, K, H, F, T, C, A, resident=True)
    check_routing(layer, ref, N, T, K, C)
    check_numerics(layer, ref, y, dx, N, T, H, E)
    x = torch.cat(pb["xs"]).cuda()
    bias = torch.from_numpy(np.concatenate(pb["biases"])).cuda()
    y2, dx2 = torch.empty_like(x), torch.empty_like(x)
    layer.forward(x, bias, T, y2)
    layer.backward(torch.cat(pb["dys"]).cuda(), dx2)
    torch.cuda.synchronize()
    assert torch.equal(y, y2) and torch.equal(dx, dx2)
    layer.close()


def test_local_first_routing_variant():
    """Opt-in local-first token routing (non-parity variant): sources hosting a
    replica keep their tokens; routing bit-exact vs the oracle's variant, numerics
    unchanged (layout-independent)."""
    N, E, K, H, F, T, C = 4, 8, 2, 256, 256, 384, 4
    pb = make_problem(N, E, K, H, F, T, 1.2, seed=21)
    A = PL.plan_layout(oracle(pb, K, PL.even_replication_layout(N, E, C), C)["routing"].R, C)
    ref = oracle(pb, K, A, C, local_first=True)
    rt = ref["routing"]
    for s_ in range(N):  # the variant's defining property
        for e in range(E):
            if A[e, s_]:
                assert rt.S[s_, e, s_] == rt.R[s_, e]
    layer, y, dx = run_gpu(pb, N, E, K, H, F, T, C, A, local_first=True)
    check_routing(layer, ref, N, T, K, C)
    check_numerics(layer, ref, y, dx, N, T, H, E)
    layer.close()
