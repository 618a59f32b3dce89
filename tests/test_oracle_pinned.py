"""Pins the planner oracle (oracle/planner_port.py) before it is trusted as a checker:
(a) the golden vectors of the reference's own unit tests, and (b) the reference
library itself (oracle/_ref) on seeded random instances."""
import json
import random

import pytest

from oracle import planner_port as P

T = P.Topology


# ---- (a) golden vectors from /root/reference/proj/tests/planner_test.cpp ----
def test_replica_allocation_goldens():
    assert P.replica_allocation([10, 10, 10, 10], 4, 4, 1) == [1, 1, 1, 1]  # :51-54
    assert P.replica_allocation([100, 10, 10, 10], 8, 4, 1) == [5, 1, 1, 1]  # :56-60
    assert P.replica_allocation([100, 10, 10, 10], 4, 4, 2) == [4, 2, 1, 1]  # :62-67
    assert P.replica_allocation([0, 0], 2, 2, 2) == [2, 2]  # :69-73
    with pytest.raises(P.PlannerError):
        P.replica_allocation([1, 1, 1], 1, 3, 2)  # :91-96
    with pytest.raises(P.PlannerError):
        P.replica_allocation([1, 1], 4, 2, 3)


def test_replica_allocation_scale_invariant():  # :75-89
    rng = random.Random(9)
    for _ in range(50):
        n = 2 + rng.randrange(6)
        c = 1 + rng.randrange(3)
        e = max(c, 1 + rng.randrange(n * c))
        loads = [float(rng.randrange(1000)) for _ in range(e)]
        assert P.replica_allocation(loads, n, e, c) == P.replica_allocation([7.0 * x for x in loads], n, e, c)


def test_expert_relocation_goldens():
    A = P.expert_relocation([1, 1], [30, 10], T(1, 2, 1e9, 1e8), 1)  # :98-104
    assert A[0][0] == 1 and A[1][1] == 1
    A = P.expert_relocation([2, 2], [10, 10], T(2, 2, 1e9, 1e8), 1)  # :106-117
    for e in range(2):
        for node in range(2):
            assert sum(A[e][d] for d in range(2 * node, 2 * node + 2)) == 1
    A = P.expert_relocation([1, 1, 2], [0, 0, 0], T(1, 2, 1e9, 1e8), 2)  # :139-148 swap repair
    assert sum(A[2]) == 2 and all(sum(A[e][d] for e in range(3)) == 2 for d in range(2))


def test_lite_routing_goldens():
    A = [[0, 1], [1, 0]]  # :175-185
    R = [[7, 0], [0, 0]]
    assert P.lite_routing(R, A, T(1, 2, 1e9, 1e8)) == [(0, 0, 1, 7)]
    A = [[0, 1, 1, 0], [1, 0, 0, 0], [0, 0, 0, 1]]  # :187-200
    R = [[5, 0, 0]] + [[0, 0, 0]] * 3
    assert P.lite_routing(R, A, T(1, 4, 1e9, 1e8)) == [(0, 0, 1, 3), (0, 0, 2, 2)]
    A = [[0, 1, 1, 1], [1, 0, 0, 0]]  # :202-214 intra-node precedence
    R = [[9, 0]] + [[0, 0]] * 3
    assert P.lite_routing(R, A, T(2, 2, 1e9, 1e8)) == [(0, 0, 1, 9)]
    A = [[0, 0, 1, 1], [1, 1, 0, 0]]  # :216-229 global fallback
    R = [[5, 0]] + [[0, 0]] * 3
    assert P.lite_routing(R, A, T(2, 2, 1e9, 1e8)) == [(0, 0, 2, 3), (0, 0, 3, 2)]


def test_static_and_even_layouts():
    A = P.static_ep_layout(4, 8, 2)  # :260-267
    for i in range(4):
        assert A[2 * i][i] == 1 and A[2 * i + 1][i] == 1
    A = P.even_replication_layout(T(1, 4, 1e9, 1e8), 4, 2)  # :278-283
    assert all(sum(row) == 2 for row in A)


def test_time_cost_golden():  # cost_test.cpp:71-88
    out = P.time_cost([(0, 0, 1, 10), (1, 0, 1, 5)], 2, T(1, 2, 100.0, 50.0), P.CostParams(1.0, 1.0, 10.0, 0))
    assert abs(out["t_comm"] - 0.4) < 1e-12 and abs(out["t_total"] - 4.9) < 1e-12
    assert out["recv"] == [0, 15]


def test_plan_layout_picks_cheaper_candidate():  # planner_test.cpp:318-345
    topo = T(1, 4, 1e9, 1e8)
    params = P.CostParams(100.0, 1e6, 1e9, 0)
    R = [[1, 22, 1]] * 4
    loads = [4.0, 88.0, 4.0]
    assert P.replica_allocation(loads, 4, 3, 1) == [1, 2, 1]
    cost = lambda reps: P.time_cost(P.lite_routing(R, P.expert_relocation(reps, loads, topo, 1), topo), 4, topo,
                                    params)["t_total"]
    chosen = P.plan_layout([R], topo, params, 1)
    got = P.time_cost(P.lite_routing(R, chosen, topo), 4, topo, params)["t_total"]
    assert got == min(cost([1, 2, 1]), cost([2, 1, 1]))


def test_lag_semantics():  # sim_test.cpp:146-179
    topo = T(1, 4, 1e9, 1e8)
    params = P.CostParams(8.0, 1e5, 1e12, 0)
    steady = [[50, 17, 17, 16]] * 4
    sentinel = [[0, 0, 0, 100]] * 4
    recs = [steady, steady, steady, sentinel]
    lay = P.lagged_layouts(recs, topo, params, 2, P.SearchSpec(), layer=0)
    expected = P.plan_layout([steady] * 3, topo, params, 2, P.SearchSpec(seed=P.mix_seed(0, 0x6C617972, 0)))
    assert lay[3] == expected


def test_mt19937_64_known_answer():
    # C++ [rand.predef]: the 10000th invocation of a default-constructed
    # mt19937_64 (seed 5489) is 9981545732273789042.
    e = P.MT19937_64(5489)
    for _ in range(9999):
        e()
    assert e() == 9981545732273789042


# ---- (b) the oracle against the reference library itself ----
def _cfg(n_nodes, dpn, c, e, eps, seed, hist="last", decay=0.5, f_ckpt=0, bi=1e9, bx=1e8):
    return json.dumps({
        "topology": {"n_nodes": n_nodes, "devices_per_node": dpn, "b_intra": bi, "b_inter": bx},
        "cost": {"v_comm": 512.0, "v_comp": 1e6, "b_comp": 1e12, "f_ckpt": f_ckpt},
        "model": {"n_experts": e, "capacity": c},
        "planner": {"epsilon": eps, "seed": seed, "history": hist, "ema_decay": decay},
    })


def test_oracle_matches_reference_library(ref, tmp_path):
    rng = random.Random(2024)
    for case in range(40):
        nodes, dpn = 1 + rng.randrange(3), 1 + rng.randrange(4)
        n = nodes * dpn
        c = 1 + rng.randrange(3)
        e = c + rng.randrange(min(16, n * c) - c + 1)
        eps = 2 + rng.randrange(4)
        seed = rng.randrange(1 << 62)
        mode = rng.choice(["last", "ema"])
        decay = rng.choice([0.25, 0.5, 0.7, 1.0])
        recs = [[[rng.randrange(60) for _ in range(e)] for _ in range(n)] for _ in range(3)]
        path = tmp_path / f"t{case}.jsonl"
        path.write_text("".join(json.dumps({"iter": t, "layer": 0, "R": recs[t]}) + "\n" for t in range(3)))
        cfg_text = _cfg(nodes, dpn, c, e, eps, seed, mode, decay)
        out = json.loads(ref.plan_layer_json(ref.config(cfg_text), ref.trace_load(str(path)), 0))
        topo = T(nodes, dpn, 1e9, 1e8)
        params = P.CostParams(512.0, 1e6, 1e12, 0)
        spec = P.SearchSpec(eps, P.mix_seed(seed, 0x6C617972, 0), mode, decay)
        for p, it in enumerate(out["iterations"]):
            A = P.plan_layout(recs[: p + 1], topo, params, c, spec)
            assert A == it["layout"], (case, p)
            if it["routing_plan"] is not None:
                ent = P.lite_routing(recs[p + 1], A, topo)
                assert [(x["src"], x["expert"], x["dst"], x["tokens"]) for x in it["routing_plan"]] == ent
                tc = P.time_cost(ent, n, topo, params)["t_total"]
                assert "%.9g" % tc == "%.9g" % it["t_total"]


def test_trace_generator_matches_reference(ref):
    spec = {"n_devices": 3, "n_experts": 5, "n_layers": 2, "n_iterations": 3, "tokens_per_device": 997,
            "skew_alpha": 0.4, "drift_sigma": 0.2, "seed": 11}
    stats = json.loads(ref.stats_json(ref.trace_generate(json.dumps(spec))))
    # Restate generate_trace (trace.cpp:89-129) for layer 0 / iteration 0.
    rng = P.Rng(P.mix_seed(11, 0x74726163, 0))
    import math
    logits = [math.log(max(rng.next_gamma(0.4), 1e-290)) for _ in range(5)]
    m = max(logits)
    ex = [math.exp(v - m) for v in logits]
    s = sum(ex)
    pop = [v / s for v in ex]
    exact = [p * 997 for p in pop]
    base = [math.floor(x) for x in exact]
    frac = sorted(((x - math.floor(x), j) for j, x in enumerate(exact)), key=lambda t: (-t[0], t[1]))
    for r in range(997 - sum(base)):
        base[frac[r % 5][1]] += 1
    rec = next(x for x in stats if x["iter"] == 0 and x["layer"] == 0)
    assert rec["expert_load"] == [3 * b for b in base]
