"""CPU checks of the layer oracle itself (no GPU): its hand-written backward
against torch autograd (float64), and the routing invariants its destination
map must satisfy (conservation vs lite routing, unique rows, segment bounds)."""
import numpy as np
import torch

from oracle import layer_oracle as LO
from oracle import planner_port as PP


def _problem(N=3, E=6, K=2, H=256, F=128, T=40, seed=0):
    rng = np.random.default_rng(seed)
    bf = lambda a: LO.bf16_round(a.astype(np.float32))
    wg = bf(rng.normal(size=(E, H)) * 0.05)
    w1 = bf(rng.normal(size=(E, F, H)) / np.sqrt(H))
    w3 = bf(rng.normal(size=(E, F, H)) / np.sqrt(H))
    w2 = bf(rng.normal(size=(E, H, F)) / np.sqrt(F))
    xs = [bf(rng.normal(size=(T, H))) for _ in range(N)]
    dys = [bf(rng.normal(size=(T, H))) for _ in range(N)]
    biases = [LO.make_bias(rng, T, E, 1.2) for _ in range(N)]
    return wg, w1, w3, w2, xs, dys, biases


def test_backward_matches_autograd():
    N, E, K, C = 3, 6, 2, 2
    wg, w1, w3, w2, xs, dys, biases = _problem(N, E, K)
    A = np.array(PP.even_replication_layout(PP.Topology(1, N, 1.0, 1.0), E, C), dtype=np.uint8)
    ref = LO.layer_step(xs, biases, wg, w1, w3, w2, K, A, C, dys)
    t = lambda a: torch.tensor(np.asarray(a), dtype=torch.float64, requires_grad=True)
    Wg, W1, W3, W2 = t(wg), t(w1), t(w3), t(w2)
    for i in range(N):
        x = t(xs[i])
        logits = x @ Wg.T + torch.tensor(biases[i], dtype=torch.float64)
        idx = torch.tensor(ref["routing"].idx[i], dtype=torch.long)
        sel = torch.gather(logits, 1, idx)
        w = torch.softmax(sel, dim=1)
        y = torch.zeros_like(x)
        for k in range(K):
            e = idx[:, k]
            g = torch.einsum("th,tfh->tf", x, W1[e])
            u = torch.einsum("th,tfh->tf", x, W3[e])
            a = torch.nn.functional.silu(g) * u
            y = y + w[:, k:k + 1] * torch.einsum("tf,thf->th", a, W2[e])
        (y * torch.tensor(dys[i], dtype=torch.float64)).sum().backward()
        assert np.allclose(y.detach().numpy(), ref["y"][i], rtol=1e-6, atol=1e-6)
        assert np.allclose(x.grad.numpy(), ref["dx"][i], rtol=1e-6, atol=1e-6)
    # expert grads accumulate over all ranks; router grad is per rank in the oracle
    assert np.allclose(W1.grad.numpy(), ref["dW1"], rtol=1e-6, atol=1e-6)
    assert np.allclose(W3.grad.numpy(), ref["dW3"], rtol=1e-6, atol=1e-6)
    assert np.allclose(W2.grad.numpy(), ref["dW2"], rtol=1e-6, atol=1e-6)
    assert np.allclose(Wg.grad.numpy(), sum(ref["dWg"]), rtol=1e-5, atol=1e-5)  # gate weights are fp32 in the oracle


def test_routing_invariants():
    for seed, (N, E, K, C) in enumerate([(8, 8, 2, 2), (4, 16, 4, 8), (2, 8, 2, 4), (8, 8, 2, 1)]):
        rng = np.random.default_rng(seed)
        T = 300
        idx = []
        for _ in range(N):
            b = LO.make_bias(rng, T, E, 1.2)
            i, _w = LO.topk(b, K)
            idx.append(i)
        R = np.stack([np.bincount(i.reshape(-1), minlength=E) for i in idx])
        A = np.array(PP.plan_layout([R.tolist()], PP.Topology(1, N, 1e9, 1e9), PP.CostParams(8.0, 1e5, 1e12), C),
                     dtype=np.uint8)
        rt = LO.route(idx, [None] * N, A, E, C)
        assert (rt.S.sum(axis=2) == rt.R).all()
        for d in range(N):
            rows = np.concatenate([rt.slot_row[i][rt.slot_dev[i] == d] for i in range(N)])
            assert len(np.unique(rows)) == len(rows)  # no two slots share a row
            total = sum(rt.seg_rows[d])
            assert len(rows) == total
            for c in range(C):
                lo, n = rt.seg_off[d, c], rt.seg_rows[d, c]
                e = rt.slot_expert[d, c]
                inseg = [(rt.slot_row[i] >= lo) & (rt.slot_row[i] < lo + n) & (rt.slot_dev[i] == d) for i in range(N)]
                assert all((idx[i][inseg[i]] == e).all() for i in range(N))
                assert sum(int(m.sum()) for m in inseg) == n


def test_router_canonical_order_is_exact_product_sum():
    """Canonical logits equal a float64 dot product up to fp32 rounding, and the
    butterfly order is what the GPU kernel documents."""
    rng = np.random.default_rng(1)
    x = LO.bf16_round(rng.normal(size=(5, 512)))
    w = LO.bf16_round(rng.normal(size=(3, 512)) * 0.05)
    lg = LO.router_logits(x, w, None)
    ref = x.astype(np.float64) @ w.astype(np.float64).T
    assert np.allclose(lg, ref, rtol=1e-5, atol=1e-5)
