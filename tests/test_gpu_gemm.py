"""Grouped tcgen05 GEMM in isolation vs a torch fp32 reference (GPU).

Tolerance: bf16 outputs with fp32 accumulation -> max|err| / max|ref| <= 1e-2;
fp32 wgrad outputs (bf16 inputs) -> <= 1e-3."""
import ctypes as C

import pytest
import torch

from paper_2602_11686_b200 import _lib

pytestmark = pytest.mark.gpu

KINDS = {"gateup": 0, "down": 1, "down_dgrad": 2, "up_dgrad": 3, "wgrad": 4}


def _fn():
    lib = _lib.load()
    f = lib.mp_fsep_debug_grouped_gemm
    ull, ll, vp, i = C.c_ulonglong, C.c_longlong, C.c_void_p, C.c_int
    f.restype = C.c_int
    f.argtypes = [i, i, vp, vp, i, i, i, vp, ull, ull, ull, vp, ull, ull, ull, ull, ull, vp, ll, ll, vp, ll, vp, ll,
                  vp]
    return f


def _run(kind, G, rows, off, M, N, K, A, a_rows, a_inner, B, b_d0, b_d1, b_groups, b_p1, b_p2, out, ldo, ogs=0,
         out2=None, ldo2=0, aux=None, ld_aux=0, pair=True, sync=True):
    f = _fn()
    st = f(KINDS[kind] | (0x100 if pair else 0), G, rows.data_ptr(), off.data_ptr(), M, N, K, A.data_ptr(), a_rows, a_inner, a_inner,
           B.data_ptr(), b_d0, b_d1, b_groups, b_p1, b_p2, out.data_ptr(), ldo, ogs,
           out2.data_ptr() if out2 is not None else None, ldo2, aux.data_ptr() if aux is not None else None, ld_aux,
           torch.cuda.current_stream().cuda_stream)
    _lib.check(st)
    if sync:
        torch.cuda.synchronize()


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-30)).item()


def _groups(counts):
    rows = torch.tensor(counts, dtype=torch.int32, device="cuda")
    off = torch.tensor([sum(counts[:g]) for g in range(len(counts))], dtype=torch.int32, device="cuda")
    return rows, off, sum(counts)


def _silu(x):
    return x * torch.sigmoid(x)


@pytest.mark.parametrize("pair", [True, False], ids=["cta_pair", "single_cta"])
@pytest.mark.parametrize("counts,H,F", [([128, 256, 0], 256, 256), ([512, 384], 1024, 512),
                                        ([256, 128, 384, 128], 2048, 1408), ([128] * 5 + [640], 512, 384)])
def test_forward_and_dgrad(counts, H, F, pair):
    torch.manual_seed(0)
    G = len(counts)
    rows, off, R = _groups(counts)
    X = (torch.randn(R, H, device="cuda") * 0.5).bfloat16()
    W13 = (torch.randn(G, 2 * F, H, device="cuda") / H ** 0.5).bfloat16()
    W2 = (torch.randn(G, H, F, device="cuda") / F ** 0.5).bfloat16()
    h = torch.empty(R, 2 * F, device="cuda", dtype=torch.bfloat16)
    act = torch.empty(R, F, device="cuda", dtype=torch.bfloat16)
    _run("gateup", G, rows, off, 0, 2 * F, H, X, R, H, W13, H, 2 * F, G, H, 2 * F * H, h, 2 * F, out2=act, ldo2=F, pair=pair)
    y = torch.empty(R, H, device="cuda", dtype=torch.bfloat16)
    _run("down", G, rows, off, 0, H, F, act, R, F, W2, F, H, G, F, H * F, y, H, pair=pair)
    dY = (torch.randn(R, H, device="cuda")).bfloat16()
    dH = torch.empty(R, 2 * F, device="cuda", dtype=torch.bfloat16)
    _run("down_dgrad", G, rows, off, 0, F, H, dY, R, H, W2, F, H, G, F, H * F, dH, 2 * F, aux=h, ld_aux=2 * F, pair=pair)
    dX = torch.empty(R, H, device="cuda", dtype=torch.bfloat16)
    _run("up_dgrad", G, rows, off, 0, H, 2 * F, dH, R, 2 * F, W13, H, 2 * F, G, H, 2 * F * H, dX, H, pair=pair)

    o = 0
    for g, c in enumerate(counts):
        if c == 0:
            continue
        sl = slice(o, o + c)
        hr = X[sl].float() @ W13[g].float().t()
        assert _rel(h[sl], hr) < 1e-2
        hb = h[sl].float().view(c, F // 128, 2, 128)
        ar = (_silu(hr.view(c, F // 128, 2, 128)[:, :, 0]) * hr.view(c, F // 128, 2, 128)[:, :, 1]).reshape(c, F)
        assert _rel(act[sl], ar) < 1e-2
        yr = act[sl].float() @ W2[g].float().t()
        assert _rel(y[sl], yr) < 1e-2
        dA = dY[sl].float() @ W2[g].float()
        gg, uu = hb[:, :, 0].reshape(c, F), hb[:, :, 1].reshape(c, F)
        sg = torch.sigmoid(gg)
        dg = dA * uu * sg * (1 + gg * (1 - sg))
        du = dA * gg * sg
        dHr = torch.stack([dg.view(c, F // 128, 128), du.view(c, F // 128, 128)], dim=2).reshape(c, 2 * F)
        assert _rel(dH[sl], dHr) < 1e-2
        dXr = dH[sl].float() @ W13[g].float()
        assert _rel(dX[sl], dXr) < 1e-2
        o += c


@pytest.mark.parametrize("pair", [True, False], ids=["cta_pair", "single_cta"])
@pytest.mark.parametrize("counts,M,N", [([128, 0, 256], 256, 512), ([384, 512], 1024, 1408), ([128, 128], 768, 256)])
def test_wgrad(counts, M, N, pair):
    torch.manual_seed(1)
    G = len(counts)
    rows, off, R = _groups(counts)
    A = torch.randn(R, M, device="cuda").bfloat16()
    B = torch.randn(R, N, device="cuda").bfloat16()
    out = torch.full((G, M, N), float("nan"), device="cuda")
    _run("wgrad", G, rows, off, M, N, 0, A, R, M, B, N, R, 1, N, 0, out, N, ogs=M * N, pair=pair)
    o = 0
    for g, c in enumerate(counts):
        ref = A[o:o + c].float().t() @ B[o:o + c].float()
        if c == 0:
            assert (out[g] == 0).all()
        else:
            assert _rel(out[g], ref) < 1e-3
        o += c


# Production-schedule wgrad launches: many tiles over several waves of the 74 CTA
# pairs.  (a) Zipf-skewed group rows: longest-processing-time group order and snake
# wave assignment (grouped_gemm2.cuh wave_tile); (b) >= 2 x 148 tiles per group, which
# turns on the wave-synchronised producers (wave_barrier) as for the Mixtral dW13.
@pytest.mark.parametrize("counts,M,N", [
    ([4096, 1920, 1152, 768, 640, 512, 384, 256, 256, 128, 128, 128, 0, 128, 384, 0], 1024, 1408),
    ([512, 1024], 8192, 2560),
], ids=["zipf_lpt_snake_5waves", "wave_sync_4waves"])
def test_wgrad_multiwave(counts, M, N):
    torch.manual_seed(2)
    G = len(counts)
    rows, off, R = _groups(counts)
    A = torch.randn(R, M, device="cuda").bfloat16()
    B = torch.randn(R, N, device="cuda").bfloat16()
    out = torch.full((G, M, N), float("nan"), device="cuda")
    _run("wgrad", G, rows, off, M, N, 0, A, R, M, B, N, R, 1, N, 0, out, N, ogs=M * N, pair=True)
    o = 0
    for g, c in enumerate(counts):
        if c == 0:
            assert (out[g] == 0).all()
        else:
            ref = A[o:o + c].float().t() @ B[o:o + c].float()
            assert _rel(out[g], ref) < 1e-3, g
        o += c
