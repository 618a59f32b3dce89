"""The exact brute-force oracle (mp_oracle_gap_json, the oracle_layout scheduler) vs the
reference library built from /root/reference (oracle/_ref): byte-identical JSON on random
tiny instances -- two-tier and single-node topologies, granularity from the gcd or the
budget, layout budgets that run out -- plus the reference's own unit-test properties
(oracle_test.cpp: exact allocation is never worse than the greedy one)."""
import json
import random

import numpy as np
import pytest

from paper_2602_11686_b200 import planner as PP


def _cfg(n, e, c, *, nodes=1, seed=3, eps=2, max_layouts=None, gran=None, f_ckpt=0):
    per = n // nodes
    d = {"topology": {"n_nodes": nodes, "devices_per_node": per, "b_intra": 9e11, "b_inter": 2e11},
         "cost": {"v_comm": 8192, "v_comp": 3.523e8, "b_comp": 1.6354e15, "f_ckpt": f_ckpt},
         "model": {"n_experts": e, "capacity": c}, "planner": {"seed": seed, "epsilon": eps}}
    if max_layouts is not None or gran is not None:
        d["oracle"] = {}
        if max_layouts is not None:
            d["oracle"]["max_layout_candidates"] = max_layouts
        if gran is not None:
            d["oracle"]["max_token_granularity"] = gran
    return json.dumps(d)


def _instances(count, rng):
    for _ in range(count):
        n = rng.choice([1, 2, 3, 4])
        c = rng.choice([1, 2])
        e = rng.randint(max(c, 1), min(4, n * c))
        if e < c:
            continue
        unit = rng.choice([1, 1, 2, 3, 8])
        R = [[unit * rng.randint(0, 20 if rng.random() < 0.3 else 6) for _ in range(e)] for _ in range(n)]
        nodes = 2 if n in (2, 4) and rng.random() < 0.5 else 1
        yield n, e, c, nodes, R


def test_oracle_gap_byte_identical_to_reference(product_lib, ref):
    rng = random.Random(17)
    checked = 0
    for n, e, c, nodes, R in _instances(160, rng):
        kw = {}
        if rng.random() < 0.15:
            kw["max_layouts"] = rng.randint(1, 6)
        cfg = _cfg(n, e, c, nodes=nodes, seed=rng.randint(0, 99), eps=rng.choice([2, 3]),
                   f_ckpt=rng.choice([0, 1]), **kw)
        inst = json.dumps({"R": R})
        try:
            theirs = ref.oracle_gap_json(ref.config(cfg), inst)
        except ref.RefError as exc:
            with pytest.raises(Exception):
                PP.oracle_gap_json(PP.Config(cfg), inst)
            continue
        mine = PP.oracle_gap_json(PP.Config(cfg), inst)
        assert mine == theirs, (cfg, inst)
        checked += 1
    assert checked > 100


def test_oracle_layout_scheduler_matches_reference(product_lib, ref, tmp_path):
    spec = json.dumps({"n_devices": 4, "n_experts": 4, "n_layers": 2, "n_iterations": 5, "tokens_per_device": 16,
                       "skew_alpha": 0.5, "drift_sigma": 0.3, "seed": 9})
    cfg = _cfg(4, 4, 2, seed=7)
    mine = PP.simulate(PP.Config(cfg), PP.Trace.generate(spec), "laer,oracle_layout,static_ep")
    theirs = ref.simulate(ref.config(cfg), ref.trace_generate(spec), "laer,oracle_layout,static_ep")
    assert mine == theirs
    rep = json.loads(mine[0])
    # the clairvoyant optimum is never beaten by the lagged greedy planner on the same iteration
    by = {}
    for r in rep["records"]:
        by.setdefault((r["iter"], r["layer"]), {})[r["scheduler"]] = r["t_total"]
    for (it, _), v in by.items():
        if it > 0:
            assert v["oracle_layout"] <= v["laer"] * (1 + 1e-9)
