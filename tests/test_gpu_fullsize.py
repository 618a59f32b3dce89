"""Full-size layer step on one B200 (Mixtral shape = BASELINE configs[1], and the fine-grained shape):
size-independent properties the oracle can afford at this size.

* routing bit-exact at full size: top-k ids vs the oracle's canonical-order router
  (numpy, all 16,384 tokens), R = bincount, per-expert segment rows;
* numerics on a random token sample: y and dx of 16 tokens vs a plain fp32 torch
  reference of the same per-token math (each token's output depends only on its
  own row, so a sample is exact), tolerance 2e-2 as everywhere;
* conservation: sum of segment rows = T*K, no receive-buffer overflow.
"""
import numpy as np
import pytest
import torch

from oracle import layer_oracle as LO
from paper_2602_11686_b200 import planner as PL
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("E,K,H,F,T", [(8, 2, 4096, 14336, 16384), (64, 8, 2048, 1408, 32768)],
                         ids=["mixtral", "fine"])
def test_full_size_properties(E, K, H, F, T):
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

    # per-token numerics on a sample, fp32 torch reference of the same math
    sample = torch.from_numpy(rng.choice(T, 16, replace=False)).cuda()
    xs, dys = x[sample].float(), dy[sample].float()
    ids = torch.from_numpy(idx_ref).cuda()[sample]
    ws = torch.from_numpy(w_ref).cuda()[sample]
    y_ref = torch.zeros_like(xs)
    dx_ref = torch.zeros_like(xs)
    dw = torch.zeros(16, K, device="cuda")
    for j in range(16):
        for k in range(K):
            e = int(ids[j, k])
            a1, a3, a2 = w1[e].float(), w3[e].float(), w2[e].float()
            gt, ut = a1 @ xs[j], a3 @ xs[j]
            sg = torch.sigmoid(gt)
            ye = a2 @ (gt * sg * ut)
            y_ref[j] += ws[j, k] * ye
            dw[j, k] = dys[j] @ ye
            da = a2.t() @ (ws[j, k] * dys[j])
            dx_ref[j] += a1.t() @ (da * ut * sg * (1 + gt * (1 - sg))) + a3.t() @ (da * gt * sg)
    # router path of dx: dl_k = w_k (dw_k - sum_j w_j dw_j), dx += sum_k dl_k wg[e_k]
    dl = ws * (dw - (ws * dw).sum(1, keepdim=True))
    for k in range(K):
        dx_ref += dl[:, k:k + 1] * wg.float()[ids[:, k]]
    assert _rel(y[sample].float(), y_ref) < 2e-2
    assert _rel(dx[sample].float(), dx_ref) < 2e-2
    layer.close()
