"""N>1 host logic on CPU with torch.distributed (gloo, world_size 2 and 4):
every rank gathers the routing histogram rows, runs the deterministic planner
on the same R and must arrive at the same layout (no broadcast needed --
SURVEY.md 8(e)), equal to the reference-pinned oracle; lite routing then gives
every rank the same send/receive counts, and the per-rank receive layout the
GPU plan kernel computes is reproduced from the gathered counts alone."""
import json
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, E, C, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    from oracle import planner_port as PP
    from paper_2602_11686_b200 import planner as PL
    cfg = json.dumps({"topology": {"n_nodes": 1, "devices_per_node": world, "b_intra": 9e11, "b_inter": 9e11},
                      "cost": {"v_comm": 8192, "v_comp": 3.523e8, "b_comp": 1.6354e15},
                      "model": {"n_experts": E, "capacity": C}, "planner": {"seed": 7}})
    planner = PL.Planner(PL.Config(cfg), world, layer=3)
    layouts = []
    hist = []
    for step in range(steps):
        A = planner.next(E)
        layouts.append(A.copy())
        rng = np.random.default_rng(1000 * step + rank)
        p = np.arange(1, E + 1) ** -1.2
        row = rng.multinomial(4096, p / p.sum()).astype(np.int64)
        rows = [torch.zeros(E, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(rows, torch.from_numpy(row))
        R = torch.stack(rows).numpy().astype(np.uint64)
        hist.append(R.astype(np.int64).tolist())
        planner.observe(R)
        S = PL.lite_routing(R, A)
        recv = S[:, :, rank].sum()
        # oracle check of the lagged layout
        topo = PP.Topology(1, world, 9e11, 9e11)
        exp = PP.even_replication_layout(topo, E, C) if step == 0 else PP.plan_layout(
            hist[:step][-1:], topo, PP.CostParams(8192, 3.523e8, 1.6354e15), C, PP.SearchSpec(2, PP.mix_seed(7, 0x6C617972, 3)))
        ok = bool(np.array_equal(A, np.array(exp, dtype=np.uint8)))
        q.put((rank, step, A.tobytes(), int(recv), ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,E,C", [(2, 8, 8), (4, 8, 4), (4, 16, 8)])
def test_ranks_agree_on_layouts(world, E, C):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, E, C, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world * 4)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    by_step = {}
    for rank, step, blob, recv, ok in out:
        assert ok, (rank, step)
        by_step.setdefault(step, set()).add(blob)
    assert all(len(v) == 1 for v in by_step.values())
