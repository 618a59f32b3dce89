"""Host-side logic of bench.py and tools/calibrate.py (CPU only): the synthetic
routing bias, the capacity rule, the token-kernel byte accounting and the
calibrated planner configuration fed to the reference `analyze` command."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import bench  # noqa: E402
import calibrate  # noqa: E402
from paper_2602_11686_b200 import planner as PL  # noqa: E402


def test_zipf_bias_marginals_follow_popularity():
    E, T, alpha = 8, 20000, 1.2
    rng = np.random.default_rng(0)
    perm = np.arange(E)
    bias = bench.zipf_bias(rng, T, E, alpha, perm)
    top1 = np.argmax(bias, axis=1)  # Gumbel-max: top-1 ~ Zipf(alpha)
    freq = np.bincount(top1, minlength=E) / T
    p = np.arange(1, E + 1, dtype=np.float64) ** -alpha
    p /= p.sum()
    assert np.abs(freq - p).max() < 0.02


def test_default_capacity_rule():
    assert bench.default_capacity(8, 2, 1) == 8          # one device holds every expert
    assert bench.default_capacity(8, 2, 4) == 4          # 2E/N
    assert bench.default_capacity(8, 2, 8) == 2
    assert bench.default_capacity(64, 8, 8) == 16
    assert bench.default_capacity(8, 2, 16) == 2         # never below top-k


class _FakeLayer:
    def __init__(self, R, A, local_first=False):
        self._R, self._A = R, A
        self.spec = type("S", (), {"local_first": local_first})()

    def histogram(self):
        return self._R

    def read(self, name):
        assert name == "layout"
        return self._A.reshape(-1)


def test_token_kernel_bytes_and_remote_rows():
    N, E, T, K, H = 2, 4, 100, 2, 256
    R = np.array([[60, 50, 50, 40], [70, 30, 50, 50]], dtype=np.uint64)
    A = np.array([[1, 1], [1, 0], [0, 1], [1, 1]], dtype=np.uint8)
    phases = {"dispatch": 0.1, "combine": 0.05, "unpermute": 0.0}
    out = bench.token_kernel_bandwidth(phases, _FakeLayer(R, A), PL, N, 0, T, K, H)
    assert set(out) == {"dispatch", "combine"}  # zero-time phases are skipped
    assert out["dispatch"]["bytes"] == T * H * 2 + T * K * H * 2
    S = PL.lite_routing(R, A)[0]
    assert out["dispatch"]["remote_rows"] == int(S.sum() - S[:, 0].sum())
    lf = bench.token_kernel_bandwidth(phases, _FakeLayer(R, A, local_first=True), PL, N, 0, T, K, H)
    # local-first keeps the tokens of experts 0, 1, 3 (hosted on rank 0) local
    assert lf["dispatch"]["remote_rows"] == int(R[0, 2])
    # shard restore: C hosted experts x (N-1)/N of 3HF bf16 parameters over the issue-to-join time
    F, C = 512, 3
    rs = bench.token_kernel_bandwidth(dict(phases, restore_ms=2.0), _FakeLayer(R, A), PL, N, 0, T, K, H, F, C)
    assert rs["restore"]["bytes"] == C * 3 * H * F * 2 * (N - 1) // N
    assert rs["restore"]["effective_GBps_per_sending_gpu"] == round(rs["restore"]["bytes"] / 2e-3 / 1e9, 1)


def test_calibrated_config_runs_reference_analysis():
    cfg = calibrate.planner_config(4, 8, 4, 2, 4096, 14336, 16384, 3.2e11, 3.1e11, 1.25e15)
    an = json.loads(PL.analyze_json(PL.Config(json.dumps(cfg))))
    # overlap_min_tokens (cost.cpp:123-143): C * bytes * b_comp / (2 * K * net_bw)
    want = int(np.ceil(4 * 2 * 1.25e15 / (2 * 2 * 3.1e11)))
    assert an["overlap"]["min_tokens_per_device"] == want
