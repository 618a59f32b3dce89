"""Real multi-GPU FSEP step (one process per GPU, CUDA IPC peer memory, barrier
kernels, attached planner) vs the CPU oracle.  Needs >= 2 GPUs; skips otherwise.
Checks per rank: top-k ids, R, layouts (lagged planner), segment sizes and every
slot's destination bit-exact; y, dx, router and expert gradients within 2e-2."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import layer_oracle as LO
from oracle import planner_port as PP

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


# the top-4 case runs the de-duplicated dispatch (one NVLink transfer per token and
# destination device) and the slot-by-slot expansion beside the gate-up GEMM
@pytest.mark.parametrize("world,E,K,H,F,T,C", [(2, 8, 2, 512, 256, 384, 4), (4, 8, 2, 256, 256, 256, 2),
                                               (4, 16, 4, 512, 256, 512, 8)])
def test_real_multi_gpu(tmp_path, world, E, K, H, F, T, C):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29517", str(ROOT / "tests" / "mp_worker.py"), str(tmp_path),
           *map(str, (E, K, H, F, T, C))]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    W = np.load(tmp_path / "weights.npz")
    topo = PP.Topology(1, world, 9e11, 9e11)
    params = PP.CostParams(2 * H, 6 * H * F, 1.6354e15)
    A = np.array(PP.even_replication_layout(topo, E, C), dtype=np.uint8)
    hist = []
    for step in range(2):
        d = [np.load(tmp_path / f"r{i}_s{step}.npz") for i in range(world)]
        for i in range(world):
            assert d[i]["barrier"][0] == 0, "barrier timeout flagged"
            assert np.array_equal(d[i]["layout"], A), (step, i)
        ref = LO.layer_step([x["x"] for x in d], [x["bias"] for x in d], W["wg"], W["w1"], W["w3"], W["w2"], K, A, C,
                            [x["dy"] for x in d])
        rt = ref["routing"]
        for i in range(world):
            assert np.array_equal(d[i]["idx"], rt.idx[i])
            assert np.array_equal(d[i]["R"], rt.R)
            assert np.array_equal(d[i]["slot"] >> 24, rt.slot_dev[i])
            assert np.array_equal(d[i]["slot"] & 0xFFFFFF, rt.slot_row[i])
            assert np.array_equal(d[i]["seg_rows"], rt.seg_rows[i])
            assert rel(d[i]["y"], ref["y"][i]) < 2e-2
            assert rel(d[i]["dx"], ref["dx"][i]) < 2e-2
            assert rel(d[i]["dwg"], ref["dWg"][i]) < 2e-2
        for name in ("dW1", "dW3", "dW2"):
            assert rel(d[0][name.lower()], ref[name]) < 2e-2, name
        hist.append(rt.R.astype(np.int64).tolist())
        A = np.array(PP.plan_layout(hist[-1:], topo, params, C, PP.SearchSpec(2, PP.mix_seed(7, 0x6C617972, 0))),
                     dtype=np.uint8)


@pytest.mark.parametrize("world", [2, 4])
def test_real_multi_gpu_modes(world):
    """Layer chaining (bit-identical to unchained), pure-EP resident experts and
    local-first routing in real multi-GPU (copy-engine) mode; see mp_worker_modes.py."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29518", str(ROOT / "tests" / "mp_worker_modes.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "modes ok" in r.stdout
