"""Wider layer shapes: non-power-of-two hidden sizes and up to 256 experts
(DeepSeek-V3-class routing: E=256, top-8, hidden 7168), run on emulated ranks with
the shipped copy-engine transport.  Routing (ids, R, every slot's destination,
segments) bit-exact vs the oracle; y, dx, router and expert gradients within 2e-2
of the torch fp32 recomputation (tests/torch_ref.py) on the oracle's routing."""
import numpy as np
import pytest
import torch

from oracle import layer_oracle as LO
from paper_2602_11686_b200 import planner as PL
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec
from test_gpu_layer import check_routing
from torch_ref import _rel, layer_ref

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,E,K,H,F,T,C", [
    (4, 256, 8, 7168, 256, 64, 64),   # DeepSeek-V3 routing and hidden size (reduced FFN and tokens)
    (2, 160, 6, 5120, 384, 96, 96),   # hidden 5120 (CH = 20), E not a power of two
    (4, 24, 2, 3072, 640, 128, 12),   # hidden 3072 (CH = 12), small E
    (2, 136, 4, 1024, 256, 100, 68),  # E > 128, not a multiple of 16: router block padded to whole warps
], ids=["e256_h7168", "e160_h5120", "e24_h3072", "e136_padded_router"])
def test_wide_shapes_copy_engine(N, E, K, H, F, T, C):
    g = torch.Generator(device="cuda").manual_seed(E + H)
    W = {e: ((torch.randn(F, H, device="cuda", generator=g) / H ** 0.5).bfloat16(),
             (torch.randn(F, H, device="cuda", generator=g) / H ** 0.5).bfloat16(),
             (torch.randn(H, F, device="cuda", generator=g) / F ** 0.5).bfloat16()) for e in range(E)}
    W["g"] = (torch.randn(E, H, device="cuda", generator=g) * 0.02).bfloat16()
    xs = [torch.randn(T, H, device="cuda", generator=g).bfloat16() for _ in range(N)]
    dys = [(torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16() for _ in range(N)]
    rng = np.random.default_rng(E)
    perm = rng.permutation(E)
    biases = [LO.make_bias(rng, T, E, 1.2, perm) for _ in range(N)]
    idx_l, w_l = [], []
    wg_np = W["g"].float().cpu().numpy()
    for v in range(N):
        i_, w_ = LO.topk(LO.router_logits(xs[v].float().cpu().numpy(), wg_np, biases[v]), K)
        idx_l.append(i_)
        w_l.append(w_)
    A = PL.plan_layout(LO.route(idx_l, w_l, PL.even_replication_layout(N, E, C), E, C).R, C)
    rt = LO.route(idx_l, w_l, A, E, C)

    layer = FsepLayer(LayerSpec(E, K, H, F, T, C, world=N, virtual=True, copy_engine=True))
    for e in range(E):
        layer.load_expert(e, *W[e])
    layer.load_router(W["g"])
    layer.set_layout(A)
    x, dy = torch.cat(xs), torch.cat(dys)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    layer.forward(x, torch.from_numpy(np.concatenate(biases)).cuda(), T, y)
    layer.backward(dy, dx)
    torch.cuda.synchronize()
    assert layer.check() == 0
    check_routing(layer, {"routing": rt}, N, T, K, C)

    errs = {}

    def on_expert(e, dW1, dW3, dW2):
        for n, a, b in zip(("dW1", "dW3", "dW2"), layer.expert_grad(e), (dW1, dW3, dW2)):
            if b.abs().max() > 0:
                errs[f"{n}[{e}]"] = _rel(a, b)

    ys, dxs, dWgs = layer_ref(xs, dys, W["g"], W.get, [torch.from_numpy(i).long().cuda() for i in idx_l],
                              [torch.from_numpy(w_).cuda() for w_ in w_l], on_expert=on_expert)
    for v in range(N):
        errs[f"y{v}"] = _rel(y[v * T:(v + 1) * T], ys[v])
        errs[f"dx{v}"] = _rel(dx[v * T:(v + 1) * T], dxs[v])
        errs[f"dWg{v}"] = _rel(layer.router_grad(v), dWgs[v])
    worst = max(errs, key=errs.get)
    assert errs[worst] < 2e-2, f"{worst}: {errs[worst]:.3e}"
    layer.close()
