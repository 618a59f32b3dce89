"""Product planner (libmoeplan_b200.so, C++ rewrite) vs the reference planner:
byte-identical JSON through the same C ABI calls, on seeded random instances and
on committed golden fixtures (tests/golden/planner_golden.json, generated from
the reference by tests/golden/make_planner_golden.py)."""
import json
import random
from pathlib import Path

import numpy as np
import pytest

from paper_2602_11686_b200 import planner as PP

GOLDEN = Path(__file__).parent / "golden" / "planner_golden.json"


def _random_case(rng: random.Random, idx: int, tmp_path: Path):
    nodes, dpn = 1 + rng.randrange(3), 1 + rng.randrange(4)
    n = nodes * dpn
    c = 1 + rng.randrange(3)
    e = c + rng.randrange(min(16, n * c) - c + 1)
    cfg = {
        "topology": {"n_nodes": nodes, "devices_per_node": dpn,
                     "b_intra": 1e9 + rng.randrange(100) * 1e9, "b_inter": 1e8 + rng.randrange(100) * 1e8},
        "cost": {"v_comm": 512.0, "v_comp": 1e6, "b_comp": 1e12, "f_ckpt": rng.randrange(2)},
        "model": {"n_experts": e, "capacity": c},
        "planner": {"epsilon": 2 + rng.randrange(4), "seed": rng.randrange(1 << 63),
                    "history": rng.choice(["last", "ema"]), "ema_decay": rng.choice([0.3, 0.5, 0.85])},
    }
    iters = 2 + rng.randrange(4)
    layers = 1 + rng.randrange(2)
    skew = rng.random() * 2.0
    lines = []
    for t in range(iters):
        for layer in range(layers):
            w = np.random.default_rng(rng.randrange(1 << 30)).zipf(1.0 + skew + 0.01, size=(n, e)) % 97
            lines.append(json.dumps({"iter": t, "layer": layer, "R": w.astype(int).tolist()}))
    path = tmp_path / f"case{idx}.jsonl"
    path.write_text("\n".join(lines) + "\n")
    return json.dumps(cfg), path, layers


def test_plan_layer_json_byte_identical(product_lib, ref, tmp_path):
    rng = random.Random(7)
    for idx in range(150):
        cfg, path, layers = _random_case(rng, idx, tmp_path)
        mine_cfg, ref_cfg = PP.Config(cfg), ref.config(cfg)
        mine_tr, ref_tr = PP.Trace.load(str(path)), ref.trace_load(str(path))
        for layer in range(layers):
            assert PP.plan_layer_json(mine_cfg, mine_tr, layer) == ref.plan_layer_json(ref_cfg, ref_tr, layer), idx


def test_simulate_byte_identical(product_lib, ref, tmp_path):
    rng = random.Random(11)
    for idx in range(40):
        cfg, path, _ = _random_case(rng, idx, tmp_path)
        a = PP.simulate(PP.Config(cfg), PP.Trace.load(str(path)), "laer,static_ep,even_replication")
        b = ref.simulate(ref.config(cfg), ref.trace_load(str(path)), "laer,static_ep,even_replication")
        assert a == b, idx


def test_generated_traces_identical(product_lib, ref):
    for seed in range(8):
        spec = json.dumps({"n_devices": 4, "n_experts": 8, "n_layers": 3, "n_iterations": 5,
                           "tokens_per_device": 4096, "skew_alpha": 0.3 + 0.2 * seed, "drift_sigma": 0.15,
                           "seed": seed})
        assert PP.Trace.generate(spec).stats_json() == ref.stats_json(ref.trace_generate(spec))


def test_analyze_identical(product_lib, ref):
    cfg = json.dumps({
        "topology": {"n_nodes": 4, "devices_per_node": 8, "b_intra": 3e11, "b_inter": 12.5e9},
        "cost": {"v_comm": 8192, "v_comp": 3.52e8, "b_comp": 312e12},
        "model": {"n_experts": 8, "capacity": 2, "p_fsep": 32, "p_ep": 4, "p_fsdp": 8,
                  "psi_expert": 352321536.0, "psi_other": 1e9, "psi_all": 4.6e10, "topk": 2},
        "planner": {"seed": 1}})
    assert PP.analyze_json(PP.Config(cfg)) == ref.analyze_json(ref.config(cfg))


def test_golden_fixtures():
    """Runs without the reference: the committed outputs of the reference planner."""
    data = json.loads(GOLDEN.read_text())
    for case in data["plan_layer"]:
        cfg = PP.Config(case["config"])
        tr = PP.Trace.generate(case["trace_spec"])
        assert PP.plan_layer_json(cfg, tr, case["layer"]) == case["output"], case["name"]
    for case in data["simulate"]:
        out = PP.simulate(PP.Config(case["config"]), PP.Trace.generate(case["trace_spec"]), case["schedulers"])
        assert out[0] == case["report"], case["name"]
    for case in data["plan_layout_arrays"]:
        A = PP.plan_layout(np.array(case["R"]), case["capacity"], bandwidth=case["bandwidth"],
                           v_comm=case["v_comm"], v_comp=case["v_comp"], b_comp=case["b_comp"],
                           seed=case["seed"])
        assert A.reshape(-1).tolist() == case["layout"], case["name"]


def test_array_api_matches_json_api(product_lib):
    """mp_fsep_plan_layout / mp_fsep_lite_routing agree with plan_layer_json."""
    rng = np.random.default_rng(5)
    n, e, c = 8, 8, 2
    R = rng.integers(0, 4000, size=(n, e))
    cfg = json.dumps({"topology": {"n_nodes": 1, "devices_per_node": n, "b_intra": 9e11, "b_inter": 9e11},
                      "cost": {"v_comm": 8192, "v_comp": 3.523e8, "b_comp": 1.6354e15},
                      "model": {"n_experts": e, "capacity": c}, "planner": {"seed": 0}})
    # plan_layer_json salts the seed per layer; the planner handle does the same.
    planner = PP.Planner(PP.Config(cfg), n, layer=0)
    planner.observe(R)
    A = planner.next(e)
    assert A.sum(axis=0).tolist() == [c] * n and (A.sum(axis=1) >= 1).all()
    S = PP.lite_routing(R, A)
    assert (S.sum(axis=2) == R).all()
    for j in range(e):
        assert ((S[:, j, :] > 0) <= (A[j][None, :] > 0)).all()


def test_error_statuses(product_lib):
    from paper_2602_11686_b200._lib import MoeplanError
    with pytest.raises(MoeplanError) as ei:
        PP.static_ep_layout(2, 5, 2)
    assert ei.value.kind == "infeasible"
    with pytest.raises(MoeplanError) as ei:
        PP.Config("{not json")
    assert ei.value.kind == "parse"
    with pytest.raises(MoeplanError) as ei:
        PP.Trace.load("/nonexistent/trace.jsonl")
    assert ei.value.kind == "io"


def test_trace_popularity_rounds_to_generated_trace(product_lib):
    """Popularity export == the shares generate_trace apportions (largest remainder)."""
    spec = json.dumps({"n_devices": 2, "n_experts": 8, "n_layers": 4, "n_iterations": 6, "tokens_per_device": 10000,
                       "skew_alpha": 0.3, "drift_sigma": 0.15, "seed": 42})
    pop = PP.trace_popularity(spec)
    assert pop.shape == (4, 6, 8) and np.allclose(pop.sum(axis=2), 1.0)
    stats = json.loads(PP.Trace.generate(spec).stats_json())
    for rec in stats:
        exact = pop[rec["layer"], rec["iter"]] * 10000
        load = np.array(rec["expert_load"]) / 2
        assert (np.abs(load - exact) < 1.0 + 1e-9).all()


def test_trace_export_replays_on_reference(product_lib, ref, tmp_path):
    """Histograms recorded through mp_fsep_trace_append save in the reference JSONL
    format; the reference library replays them to byte-identical reports."""
    rng = np.random.default_rng(3)
    tr = PP.Trace.create(4, 8)
    for it in range(5):
        for layer in (0, 1):
            p = np.arange(1, 9) ** -1.2
            tr.append(it, layer, np.stack([rng.multinomial(2048, p / p.sum()) for _ in range(4)]))
    path = tmp_path / "observed.jsonl"
    tr.save(str(path))
    assert PP.Trace.load(str(path)).dims() == (4, 8, 10)
    cfg = json.dumps({"topology": {"n_nodes": 1, "devices_per_node": 4, "b_intra": 9e11, "b_inter": 9e11},
                      "cost": {"v_comm": 8192, "v_comp": 3.523e8, "b_comp": 1.6354e15},
                      "model": {"n_experts": 8, "capacity": 4}, "planner": {"seed": 7}})
    mine = PP.simulate(PP.Config(cfg), PP.Trace.load(str(path)), "laer,static_ep")
    theirs = ref.simulate(ref.config(cfg), ref.trace_load(str(path)), "laer,static_ep")
    assert mine == theirs
    from paper_2602_11686_b200._lib import MoeplanError
    with pytest.raises(MoeplanError):
        tr.append(0, 0, np.zeros((4, 8)))  # duplicate (iter, layer)


def test_plan_next_matches_planner_handle_and_port(product_lib):
    """mp_fsep_plan_next == a planner handle after one observation ==
    the pinned port's plan_layout([R]) with the layer-salted seed, for several layers."""
    rng = np.random.default_rng(11)
    n, e, c = 8, 16, 4
    cfg_json = json.dumps({"topology": {"n_nodes": 1, "devices_per_node": n, "b_intra": 9e11, "b_inter": 9e11},
                           "cost": {"v_comm": 4096, "v_comp": 1.73e7, "b_comp": 1.6354e15},
                           "model": {"n_experts": e, "capacity": c}, "planner": {"seed": 5, "epsilon": 4}})
    cfg = PP.Config(cfg_json)
    from oracle import planner_port as PORT
    topo = PORT.Topology(1, n, 9e11, 9e11)
    params = PORT.CostParams(4096, 1.73e7, 1.6354e15)
    for layer in range(3):
        R = rng.integers(0, 5000, size=(n, e))
        A = PP.plan_next(cfg, R, layer)
        h = PP.Planner(cfg, n, layer)
        h.observe(R)
        assert np.array_equal(A, h.next(e))
        want = PORT.plan_layout([R.astype(np.int64).tolist()], topo, params, c,
                                PORT.SearchSpec(4, PORT.mix_seed(5, 0x6C617972, layer)))
        assert np.array_equal(A, np.array(want, dtype=np.uint8))


@pytest.mark.parametrize("nodes,dpn,e,c", [(8, 8, 128, 2), (16, 8, 256, 4), (4, 8, 64, 8), (1, 72, 256, 4), (128, 8, 1024, 2)])
def test_large_instances_byte_identical(product_lib, ref, tmp_path, nodes, dpn, e, c):
    """Cluster-scale instances (64-1024 devices, up to 1024 experts; the relocation's node
    balancing and repair paths get exercised far more than at <= 12 devices)."""
    n = nodes * dpn
    rng = np.random.default_rng(n * 1000 + e + c)
    cfg = json.dumps({
        "topology": {"n_nodes": nodes, "devices_per_node": dpn, "b_intra": 9e11, "b_inter": 5e10},
        "cost": {"v_comm": 8192.0, "v_comp": 3.52e8, "b_comp": 1.6354e15, "f_ckpt": 0},
        "model": {"n_experts": e, "capacity": c},
        "planner": {"epsilon": 3, "seed": int(rng.integers(1 << 62)), "history": "ema", "ema_decay": 0.5},
    })
    lines = []
    for t in range(3):
        p = rng.permutation(e)
        w = (np.arange(1, e + 1, dtype=np.float64) ** -1.2)[p]
        R = np.stack([rng.multinomial(4096 * 8, w / w.sum()) for _ in range(n)])
        lines.append(json.dumps({"iter": t, "layer": 0, "R": R.astype(int).tolist()}))
    path = tmp_path / "large.jsonl"
    path.write_text("\n".join(lines) + "\n")
    mine = PP.plan_layer_json(PP.Config(cfg), PP.Trace.load(str(path)), 0)
    theirs = ref.plan_layer_json(ref.config(cfg), ref.trace_load(str(path)), 0)
    assert mine == theirs


def test_20k_instance_hash_matches_reference(product_lib):
    """oracle/planner_hash.cpp, one source written against the shared
    C++ API, built against the reference objects (oracle/build_ref.sh) and against this
    library; plan_layout + lite_routing + time_cost over 20,000 seeded random instances
    (1-32 devices, 1-4 nodes, up to 64 experts, 1-3 history steps, last / EMA, epsilon
    2-5) must hash identically."""
    import subprocess
    root = Path(__file__).resolve().parents[1]
    ref_bin = root / "oracle" / "_ref" / "planner_hash_ref"
    if not ref_bin.exists():
        pytest.skip("reference planner_hash not built (reference tree absent)")
    src = root / "oracle" / "planner_hash.cpp"
    lib = root / "paper_2602_11686_b200" / "lib"
    ours = root / "oracle" / "_ref" / "planner_hash_b200"
    if not ours.exists() or ours.stat().st_mtime < max(src.stat().st_mtime, (lib / "libmoeplan_b200.so").stat().st_mtime):
        subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{root / 'include'}", str(src),
                        f"-L{lib}", "-l:libmoeplan_b200.so", f"-Wl,-rpath,{lib}", "-o", str(ours)], check=True)
    a = subprocess.run([str(ref_bin), "20000", "1"], capture_output=True, text=True, check=True).stdout.split()
    b = subprocess.run([str(ours), "20000", "1"], capture_output=True, text=True, check=True).stdout.split()
    assert a[0] == "20000" and a == b, (a, b)
