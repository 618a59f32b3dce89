"""Seeded random layer shapes on emulated ranks vs the oracle: world sizes 1-8 (incl. 3,
5 and 6) plus the 16-rank maximum, top-k 1-8, ragged token counts (not multiples of the
64-token router tile), hidden sizes from the supported set, capacities from the minimum
(E/N) to full replication, planned or static layouts, and both transports (device kernels / the shipped copy-engine
path).  Routing bit-exact; y, dx, router and expert gradients within 2e-2."""
import random

import numpy as np
import pytest

from paper_2602_11686_b200 import planner as PL
from test_gpu_layer import check_numerics, check_routing, make_problem, oracle, run_gpu

pytestmark = pytest.mark.gpu


def _cases(n):
    rng = random.Random(2602)
    out = []
    while len(out) < n:
        N = rng.choice([1, 2, 3, 4, 5, 6, 8, 8])
        E = rng.choice([8, 16, 24, 32])
        K = rng.choice([k for k in (1, 2, 3, 4, 6, 8) if k <= E])
        H = rng.choice([256, 512, 768, 1280])
        F = rng.choice([128, 256, 384])
        if (3 * H * F) % (8 * N):
            continue
        c_min = max(K if N == 1 else 1, -(-E // N))
        C = E if N == 1 else rng.randint(max(c_min, min(K, E)), E)
        if K > C * N:
            continue
        T = rng.choice([1, 37, 100, 129, 257])
        layout = rng.choice(["planned", "static", "even"]) if N > 1 else "even"
        ce = N > 1 and rng.random() < 0.6
        out.append((N, E, K, H, F, T, C, layout, ce))
    return out


# plus the largest world the runtime supports (16 ranks) on both transports
_EXTRA = [(16, 32, 4, 256, 128, 64, 2, "planned", True), (16, 48, 6, 512, 256, 33, 4, "static", False)]


@pytest.mark.parametrize("N,E,K,H,F,T,C,layout,ce", _cases(16) + _EXTRA)
def test_random_shape(N, E, K, H, F, T, C, layout, ce):
    pb = make_problem(N, E, K, H, F, T, 1.1, seed=N * 1000 + E * 10 + K)
    if layout == "static":
        A = PL.static_ep_layout(N, E, C)
    elif layout == "planned":
        A = PL.plan_layout(oracle(pb, K, PL.even_replication_layout(N, E, C), C)["routing"].R, C)
    else:
        A = PL.even_replication_layout(N, E, C)
    ref = oracle(pb, K, A, C)
    layer, y, dx = run_gpu(pb, N, E, K, H, F, T, C, A, copy_engine=ce)
    assert layer.check() == 0
    check_routing(layer, ref, N, T, K, C)
    check_numerics(layer, ref, y, dx, N, T, H, E)
    layer.close()
