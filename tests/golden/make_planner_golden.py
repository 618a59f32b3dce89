"""Generates tests/golden/planner_golden.json from the REFERENCE planner
(oracle/_ref, built from /root/reference/proj/src).  Run in the build
container: python tests/golden/make_planner_golden.py"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402


def cfg(n, e, c, seed, eps=2, hist="last", bw=9e11, v_comm=8192.0, v_comp=3.523e8, b_comp=1.6354e15):
    return json.dumps({"topology": {"n_nodes": 1, "devices_per_node": n, "b_intra": bw, "b_inter": bw},
                       "cost": {"v_comm": v_comm, "v_comp": v_comp, "b_comp": b_comp},
                       "model": {"n_experts": e, "capacity": c},
                       "planner": {"epsilon": eps, "seed": seed, "history": hist}})


def main():
    assert ref.available(), "needs the reference library"
    out = {"plan_layer": [], "simulate": [], "plan_layout_arrays": []}
    cases = [
        # name, N, E, C, tokens, alpha, sigma, eps, hist
        ("mixtral_e8_n8_c2", 8, 8, 2, 32768, 0.3, 0.15, 2, "last"),
        ("mixtral_e8_n4_c4", 4, 8, 4, 32768, 1.0, 0.15, 3, "last"),
        ("fine_e64_n8_c16", 8, 64, 16, 262144, 0.5, 0.15, 2, "last"),
        ("tiny_e8_n8_c2_ema", 8, 8, 2, 1024, 0.3, 0.3, 4, "ema"),
        ("n2_e8_c4", 2, 8, 4, 32768, 0.3, 0.15, 2, "last"),
    ]
    for name, n, e, c, tok, alpha, sigma, eps, hist in cases:
        spec = json.dumps({"n_devices": n, "n_experts": e, "n_layers": 2, "n_iterations": 4,
                           "tokens_per_device": tok, "skew_alpha": alpha, "drift_sigma": sigma, "seed": 42})
        conf = cfg(n, e, c, 7, eps, hist)
        rc, rt = ref.config(conf), ref.trace_generate(spec)
        out["plan_layer"].append({"name": name, "config": conf, "trace_spec": spec, "layer": 1,
                                  "output": ref.plan_layer_json(rc, rt, 1)})
        rep, _ = ref.simulate(rc, rt, "laer,static_ep,even_replication")
        out["simulate"].append({"name": name, "config": conf, "trace_spec": spec,
                                "schedulers": "laer,static_ep,even_replication", "report": rep})
    import numpy as np
    rng = np.random.default_rng(3)
    for k, (n, e, c) in enumerate([(8, 8, 2), (8, 64, 16), (4, 8, 4), (8, 8, 1), (2, 8, 4)]):
        p = np.arange(1, e + 1) ** -1.2
        R = np.stack([rng.multinomial(4096, p / p.sum()) for _ in range(n)])
        res = ref.plan_bench(R.tolist(), c, 1, bandwidth=9e11, v_comm=8192.0, v_comp=3.523e8, b_comp=1.6354e15,
                             seed=k)
        out["plan_layout_arrays"].append({"name": f"zipf_{n}_{e}_{c}", "R": R.tolist(), "capacity": c,
                                          "bandwidth": 9e11, "v_comm": 8192.0, "v_comp": 3.523e8,
                                          "b_comp": 1.6354e15, "seed": k, "layout": res["layout"]})
    (Path(__file__).parent / "planner_golden.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
