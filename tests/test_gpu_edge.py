"""Edge cases of the GPU layer step: empty and single-token batches, bitwise
determinism across repeated steps, CUDA-graph replay == eager, and the
histogram/layout bookkeeping when most experts receive nothing."""
import numpy as np
import pytest
import torch

from paper_2602_11686_b200._lib import MoeplanError

from oracle import layer_oracle as LO
from paper_2602_11686_b200 import planner as PL
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec

pytestmark = pytest.mark.gpu


def _layer(N, E, K, H, F, T, C, seed=0, max_recv_rows=0):
    g = torch.Generator().manual_seed(seed)
    layer = FsepLayer(LayerSpec(E, K, H, F, T, C, world=N, virtual=True, max_recv_rows=max_recv_rows))
    w = {}
    for e in range(E):
        w1 = (torch.randn(F, H, generator=g) / H ** 0.5).bfloat16().cuda()
        w3 = (torch.randn(F, H, generator=g) / H ** 0.5).bfloat16().cuda()
        w2 = (torch.randn(H, F, generator=g) / F ** 0.5).bfloat16().cuda()
        layer.load_expert(e, w1, w3, w2)
    layer.load_router((torch.randn(E, H, generator=g) * 0.02).bfloat16().cuda())
    return layer


def _inputs(N, T, H, E, alpha, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(N * T, H, generator=g).bfloat16().cuda()
    dy = (torch.randn(N * T, H, generator=g) * 0.1).bfloat16().cuda()
    rng = np.random.default_rng(seed)
    bias = torch.from_numpy(np.concatenate([LO.make_bias(rng, T, E, alpha) for _ in range(N)])).cuda()
    return x, dy, bias


def test_empty_and_single_token_batches():
    N, E, K, H, F, T, C = 2, 8, 2, 256, 256, 128, 4
    layer = _layer(N, E, K, H, F, T, C)
    for n in (0, 1):
        x, dy, bias = _inputs(N, max(n, 1), H, E, 1.0, 3)
        y = torch.zeros_like(x)
        dx = torch.zeros_like(x)
        layer.forward(x, bias, n, y)
        layer.backward(dy, dx)
        torch.cuda.synchronize()
        R = layer.histogram()
        assert R.sum() == N * n * K
        dw1, dw3, dw2 = layer.expert_grad(0)
        torch.cuda.synchronize()
        assert torch.isfinite(dw1).all() and torch.isfinite(dw2).all()
        if n == 0:
            assert float(dw1.abs().max()) == 0.0 and float(layer.router_grad(0).abs().max()) == 0.0
    layer.close()


@pytest.mark.parametrize("E,K,C", [(8, 2, 4), (16, 4, 8)], ids=["top2", "top4_dedupe"])
def test_bitwise_determinism_and_graph_replay(E, K, C):
    """Eager steps reproduce bit for bit; a captured CUDA graph replays them (top-4:
    with the de-duplicated token transfers and their expansion kernels)."""
    N, H, F, T = 4, 512, 384, 256
    layer = _layer(N, E, K, H, F, T, C, seed=1)
    x, dy, bias = _inputs(N, T, H, E, 1.2, 5)
    outs = []
    for _ in range(2):
        y = torch.empty_like(x)
        dx = torch.empty_like(x)
        layer.forward(x, bias, T, y)
        layer.backward(dy, dx)
        torch.cuda.synchronize()
        outs.append((y.clone(), dx.clone(), layer.expert_grad(3)[0].clone(), layer.router_grad(1).clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b), "eager steps are not bitwise reproducible"
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    layer.graph_step(x, bias, T, y, dy, dx)
    layer.graph_step(x, bias, T, y, dy, dx)  # replay of the captured graph
    torch.cuda.synchronize()
    assert torch.equal(y, outs[0][0]) and torch.equal(dx, outs[0][1])
    assert torch.equal(layer.expert_grad(3)[0], outs[0][2])
    layer.close()


def test_extreme_skew_most_experts_idle():
    """Zipf 3.0 over 16 experts, top-1: most experts get no tokens at all."""
    N, E, K, H, F, T, C = 2, 16, 1, 256, 256, 256, 8
    layer = _layer(N, E, K, H, F, T, C, seed=2)
    x, dy, bias = _inputs(N, T, H, E, 3.0, 9)
    A = PL.even_replication_layout(N, E, C)
    layer.set_layout(A)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    layer.forward(x, bias, T, y)
    layer.backward(dy, dx)
    torch.cuda.synchronize()
    R = layer.histogram()
    assert (R.sum(axis=0) == 0).sum() >= 4
    assert R.sum() == N * T * K
    for v in range(N):
        seg = layer.read("seg_rows", v).view(np.int32)
        assert seg.sum() == layer.read("total_rows", v).view(np.int32)[0] - (
            (-seg) % 128).sum()  # padded total == sum of padded segments
    assert torch.isfinite(y.float()).all() and torch.isfinite(dx.float()).all()
    layer.close()


def test_receive_overflow_is_flagged_and_memory_safe():
    """An undersized receive buffer (max_recv_rows) flags status=1 and drops the
    segments that do not fit -- no out-of-bounds writes: the device stays healthy
    and a correctly sized layer afterwards still matches its own eager rerun."""
    N, E, K, H, F, T, C = 2, 8, 2, 256, 256, 512, 8
    small = _layer(N, E, K, H, F, T, C, max_recv_rows=256)
    small.set_layout(PL.even_replication_layout(N, E, C))
    x, dy, bias = _inputs(N, T, H, E, 1.5, seed=3)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    small.forward(x, bias, T, y)
    torch.cuda.synchronize()
    assert any(small.read("status", v).view(np.int32)[0] == 1 for v in range(N))
    with pytest.raises(MoeplanError) as ei:  # loud: the failed step is reported (MP_ERR_DEVICE)
        small.backward(dy, dx)
    assert ei.value.status == 7
    small.close()
    ok = _layer(N, E, K, H, F, T, C)
    ok.set_layout(PL.even_replication_layout(N, E, C))
    outs = []
    for _ in range(2):
        y, dx = torch.empty_like(x), torch.empty_like(x)
        ok.forward(x, bias, T, y)
        ok.backward(dy, dx)
        torch.cuda.synchronize()
        outs.append((y.clone(), dx.clone()))
    assert all(ok.read("status", v).view(np.int32)[0] == 0 for v in range(N))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    ok.close()
