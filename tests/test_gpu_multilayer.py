"""4 stacked FSEP layers on one GPU (8 -> 4 emulated ranks), the shipped multi-GPU transport
(MP_FSEP_FLAG_COPY_ENGINE), drifting per-iteration routing and a planner per layer that
re-lays the experts out every step -- BASELINE configs[3] at reduced shapes -- checked
layer by layer, step by step, against the oracle.

* Chained layers (mp_fsep_layer_chain, PAPER Fig.5): layer l+1's shard restore is issued
  after layer l's gate-up GEMM and overlaps layer l's down GEMM / combine and layer
  l+1's router and dispatch.
* With defer_rs (PAPER Fig.5(e)) layer l+1's gradient reduce-scatter
  completes on a side stream under layer l's backward GEMMs.
* Per-layer lag and seeds as the reference simulator (sim.cpp:108-131): step 0 of every
  layer runs on the even-replication layout, step t on plan_layout(R_0..R_{t-1}) with
  seed mix_seed(seed, "layr", layer).
Each layer is checked on the inputs it actually received (the previous layer's GPU
output in the forward, the next layer's GPU dx in the backward): routing, R, layouts,
segments and every slot's destination bit-exact; y, dx, router and expert gradients
within 2e-2.
"""
import json

import numpy as np
import pytest
import torch

from oracle import layer_oracle as LO
from oracle import planner_port as PP
from paper_2602_11686_b200 import planner as PL
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec
from test_gpu_layer import check_numerics, check_routing

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("defer_rs", [False, True], ids=["rs_in_layer", "rs_deferred"])
def test_four_chained_layers_drifting_routing(defer_rs):
    N, E, K, H, F, T, C, NL, STEPS = 4, 8, 2, 256, 256, 256, 3, 4, 3
    g = torch.Generator().manual_seed(77)
    W = []
    layers = []
    cfg = PL.Config(json.dumps({"topology": {"n_nodes": 1, "devices_per_node": N, "b_intra": 9e11, "b_inter": 9e11},
                                "cost": {"v_comm": 2 * H, "v_comp": 6 * H * F, "b_comp": 1.6354e15},
                                "model": {"n_experts": E, "capacity": C}, "planner": {"seed": 7}}))
    for l in range(NL):
        w = dict(wg=(torch.randn(E, H, generator=g) * 0.02).bfloat16(),
                 w1=(torch.randn(E, F, H, generator=g) / H ** 0.5).bfloat16(),
                 w3=(torch.randn(E, F, H, generator=g) / H ** 0.5).bfloat16(),
                 w2=(torch.randn(E, H, F, generator=g) / F ** 0.5).bfloat16())
        W.append(w)
        layer = FsepLayer(LayerSpec(E, K, H, F, T, C, world=N, virtual=True, copy_engine=True, defer_rs=defer_rs))
        for e in range(E):
            layer.load_expert(e, w["w1"][e].cuda().contiguous(), w["w3"][e].cuda().contiguous(),
                              w["w2"][e].cuda().contiguous())
        layer.load_router(w["wg"].cuda())
        layer.attach_planner(cfg, layer=l)
        layers.append(layer)
    for l in range(NL - 1):
        layers[l].chain(layers[l + 1])
    spec = json.dumps({"n_devices": N, "n_experts": E, "n_layers": NL, "n_iterations": STEPS,
                       "tokens_per_device": T, "skew_alpha": 0.3, "drift_sigma": 0.15, "seed": 42})
    logp = np.log(np.maximum(PL.trace_popularity(spec), 1e-30))
    rng = np.random.default_rng(5)
    x = torch.randn(N * T, H, generator=g).bfloat16().cuda()
    dy = (torch.randn(N * T, H, generator=g) * 0.1).bfloat16().cuda()
    ys = [torch.empty_like(x) for _ in range(NL)]
    dxs = [torch.empty_like(x) for _ in range(NL)]
    topo = PP.Topology(1, N, 9e11, 9e11)
    params = PP.CostParams(2 * H, 6 * H * F, 1.6354e15)
    history = [[] for _ in range(NL)]
    A = [np.array(PP.even_replication_layout(topo, E, C), dtype=np.uint8) for _ in range(NL)]
    changed = 0
    for step in range(STEPS):
        biases = [[(logp[l, step][None, :] + rng.gumbel(size=(T, E))).astype(np.float32) for _ in range(N)]
                  for l in range(NL)]
        h = x
        for l in range(NL):
            layers[l].forward(h, torch.from_numpy(np.concatenate(biases[l])).cuda(), T, ys[l])
            h = ys[l]
        gr = dy
        for l in reversed(range(NL)):
            layers[l].backward(gr, dxs[l])
            gr = dxs[l]
        torch.cuda.synchronize()
        for l in range(NL):
            assert layers[l].check() == 0
            assert np.array_equal(layers[l].read("layout", 0).reshape(E, N), A[l]), (step, l)
            xin = (x if l == 0 else ys[l - 1]).float().cpu().numpy().reshape(N, T, H)
            din = (dy if l == NL - 1 else dxs[l + 1]).float().cpu().numpy().reshape(N, T, H)
            f32 = lambda t: t.float().numpy()
            ref = LO.layer_step(list(xin), biases[l], f32(W[l]["wg"]), f32(W[l]["w1"]), f32(W[l]["w3"]),
                                f32(W[l]["w2"]), K, A[l], C, list(din))
            check_routing(layers[l], ref, N, T, K, C)
            check_numerics(layers[l], ref, ys[l], dxs[l], N, T, H, E)
            history[l].append(layers[l].histogram().astype(np.int64).tolist())
            nxt = np.array(PP.plan_layout(history[l], topo, params, C, PP.SearchSpec(2, PP.mix_seed(7, 0x6C617972, l))),
                           dtype=np.uint8)
            changed += int(not np.array_equal(nxt, A[l]))
            A[l] = nxt
    assert changed > 0, "the planners never re-laid out any layer"
    for layer in layers:
        layer.close()
