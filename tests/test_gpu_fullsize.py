"""Full-size layer step on one B200 (Mixtral shape = BASELINE configs[1], and the fine-grained
shape configs[2]), checked in full against the oracle's routing and a torch fp32 reference.

* routing bit-exact at full size: top-k ids vs the oracle's canonical-order router
  (numpy, every token), R = bincount, per-expert segment rows, conservation
  (sum of segment rows = T*K), no receive-buffer overflow;
* numerics in full, tolerance max|gpu - ref| / max|ref| <= 2e-2 (north star):
  y and dx of every token, the router gradient dWg, and dW1 / dW3 / dW2 of every
  expert -- the production multi-wave wgrad launches (Mixtral dW13: 112 x 16 tiles
  per expert over ~24 waves; LPT group order, snake waves and wave barriers) --
  against tests/torch_ref.py (fp32 torch recomputation of layer_oracle.layer_step
  from the oracle's routing).
"""
import numpy as np
import pytest
import torch

from oracle import layer_oracle as LO
from paper_2602_11686_b200 import planner as PL
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec
from torch_ref import _rel, layer_ref

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.mark.parametrize("E,K,H,F,T", [(8, 2, 4096, 14336, 16384), (64, 8, 2048, 1408, 32768)],
                         ids=["mixtral", "fine"])
def test_full_size_parity(E, K, H, F, T):
    g = torch.Generator(device="cuda").manual_seed(42)
    wg = (torch.randn(E, H, device="cuda", generator=g) * 0.02).bfloat16()
    w1 = [(torch.randn(F, H, device="cuda", generator=g) / H ** 0.5).bfloat16() for _ in range(E)]
    w3 = [(torch.randn(F, H, device="cuda", generator=g) / H ** 0.5).bfloat16() for _ in range(E)]
    w2 = [(torch.randn(H, F, device="cuda", generator=g) / F ** 0.5).bfloat16() for _ in range(E)]
    x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    dy = (torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16()
    rng = np.random.default_rng(7)
    bias = LO.make_bias(rng, T, E, 1.2, rng.permutation(E))
    layer = FsepLayer(LayerSpec(E, K, H, F, T, E, world=1))
    for e in range(E):
        layer.load_expert(e, w1[e], w3[e], w2[e])
    layer.load_router(wg)
    layer.set_layout(PL.even_replication_layout(1, E, E))
    y, dx = torch.empty_like(x), torch.empty_like(x)
    bias_d = torch.from_numpy(bias).cuda()
    layer.forward(x, bias_d, T, y)
    layer.backward(dy, dx)
    torch.cuda.synchronize()
    assert layer.check() == 0

    # routing, bit-exact at full size
    logits = LO.router_logits(x.float().cpu().numpy(), wg.float().cpu().numpy(), bias)
    idx_ref, w_ref = LO.topk(logits, K)
    idx = layer.read("topk_idx").view(np.int32).reshape(T, K)
    assert np.array_equal(idx, idx_ref)
    counts = np.bincount(idx_ref.reshape(-1), minlength=E)
    assert np.array_equal(layer.histogram()[0], counts)
    seg = layer.read("seg_rows").view(np.int32)
    assert np.array_equal(seg, counts) and seg.sum() == T * K
    assert layer.read("status").view(np.int32)[0] == 0
    w_gpu = layer.read("topk_w").view(np.float32).reshape(T, K)
    assert np.abs(w_gpu - w_ref).max() < 1e-5

    # numerics in full vs the fp32 torch reference (oracle routing)
    errs = {}

    def on_expert(e, dW1, dW3, dW2):
        g1, g3, g2 = layer.expert_grad(e)
        errs[f"dW1[{e}]"] = _rel(g1, dW1)
        errs[f"dW3[{e}]"] = _rel(g3, dW3)
        errs[f"dW2[{e}]"] = _rel(g2, dW2)

    ys, dxs, dWgs = layer_ref([x], [dy], wg, lambda e: (w1[e], w3[e], w2[e]),
                              [torch.from_numpy(idx_ref).long().cuda()], [torch.from_numpy(w_ref).cuda()],
                              on_expert=on_expert)
    errs["y"] = _rel(y, ys[0])
    errs["dx"] = _rel(dx, dxs[0])
    errs["dWg"] = _rel(layer.router_grad(0), dWgs[0])
    worst = max(errs, key=errs.get)
    print(f"\nfull-size parity {E}x{H}x{F}: worst {worst} {errs[worst]:.3e}; y {errs['y']:.3e} dx {errs['dx']:.3e} "
          f"dWg {errs['dWg']:.3e}")
    assert errs[worst] < TOL, f"{worst}: {errs[worst]:.3e}  (all: {errs})"
    layer.close()
