"""B200-calibrated planner cost parameters.

Reads bench JSON lines measured on the pool (N>1 runs carry per-phase and
token-kernel timings) and derives the rates the reference cost model takes:

  b_comp   achieved grouped-GEMM TFLOP/s of the expert FFN   (CostParams.b_comp)
  b_intra  achieved NVLink rate of the token dispatch A2A    (Topology link bandwidth)
  b_inter  copy-engine push rate of the shard restore        (network bandwidth of the
           prefetch-overlap analysis, overlap_min_tokens, cost.cpp:123-143)

It then runs the reference `analyze` command (mp_analyze_json, byte-compatible)
with nominal and calibrated rates, reports min_tokens_per_device for which the
expert-granular restore hides under the FFN compute, and checks that against the
measured runs (forward GEMM time vs half the backward GEMM time: a stalled
restore shows up as a forward/backward ratio above 0.5).

  python tools/calibrate.py profiles/r01_bench_n4_mixtral_full.json ... \
      [--restore-gbps 310] [--out profiles/b200_calibration.json]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def last_json(path: Path) -> dict:
    lines = [l for l in path.read_text().splitlines() if l.startswith("{")]
    return json.loads(lines[-1])


def planner_config(N, E, C, K, H, F, T, b_intra, b_inter, b_comp):
    return {"topology": {"n_nodes": 1, "devices_per_node": N, "b_intra": b_intra, "b_inter": b_inter},
            "cost": {"v_comm": 2.0 * H, "v_comp": 6.0 * H * F, "b_comp": b_comp},
            "model": {"n_experts": E, "capacity": C, "p_fsep": N, "p_ep": max(1, N // 2), "p_fsdp": N // max(1, N // 2),
                      "psi_expert": 3.0 * H * F * 2, "hidden": H, "intermediate": F, "topk": K,
                      "tokens_per_device": T, "bytes_per_element": 2},
            "planner": {"seed": 7}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("runs", nargs="+")
    ap.add_argument("--restore-gbps", type=float, default=310.0,
                    help="copy-engine push rate per GPU (tools/ce_probe.py; DESIGN.md section 4)")
    ap.add_argument("--out", default=str(ROOT / "profiles" / "b200_calibration.json"))
    args = ap.parse_args()
    from paper_2602_11686_b200 import planner as PL

    runs = [last_json(Path(p)) for p in args.runs]
    out = {"runs": [], "configs": {}}
    by_shape = {}
    for p, d in zip(args.runs, runs):
        c = d["config"]
        tk = d.get("token_kernels_layer0") or {}
        pr = d.get("phases_ms_per_rank_layer0") or {}
        rec = {"file": p, "workload": c["workload"], "n_gpus": d["n_gpus"], "gemm_tflops": d["roofline"]["achieved"],
               "dispatch_nvlink_GBps": (tk.get("dispatch") or {}).get("nvlink_GBps"),
               "fwd_over_half_bwd_gemm": [round(f / (b / 2), 3) for f, b in zip(pr.get("fwd_gemms", []),
                                                                                pr.get("bwd_gemms", []))]}
        out["runs"].append(rec)
        key = (c["n_experts"], c["top_k"], c["hidden"], c["ffn"], c["tokens_per_gpu"], c["capacity"], d["n_gpus"])
        by_shape.setdefault(key, []).append(rec)
    for (E, K, H, F, T, C, N), recs in by_shape.items():
        b_comp = statistics.median(r["gemm_tflops"] for r in recs) * 1e12
        nv = [r["dispatch_nvlink_GBps"] for r in recs if r["dispatch_nvlink_GBps"]]
        b_intra = statistics.median(nv) * 1e9 if nv else 9e11
        b_inter = args.restore_gbps * 1e9
        res = {}
        for name, cfg in (("nominal", planner_config(N, E, C, K, H, F, T, 9e11, 9e11, 1.6354e15)),
                          ("calibrated", planner_config(N, E, C, K, H, F, T, b_intra, b_inter, b_comp))):
            an = json.loads(PL.analyze_json(PL.Config(json.dumps(cfg))))
            res[name] = {"planner_config": cfg, "analysis": an,
                         "restore_hidden_predicted": T >= an["overlap"]["min_tokens_per_device"]}
        ratios = [x for r in recs for x in r["fwd_over_half_bwd_gemm"]]
        res["measured"] = {"b_comp": b_comp, "b_intra": b_intra, "b_inter": b_inter, "tokens_per_device": T,
                           "fwd_over_half_bwd_gemm": ratios,
                           "restore_hidden_measured": bool(ratios) and max(ratios) <= 1.05}
        out["configs"][f"E{E}_K{K}_H{H}_F{F}_T{T}_C{C}_N{N}"] = res
    Path(args.out).write_text(json.dumps(out, indent=1))
    for k, v in out["configs"].items():
        print(k, "min tokens/device: nominal", v["nominal"]["analysis"]["overlap"]["min_tokens_per_device"],
              "calibrated", v["calibrated"]["analysis"]["overlap"]["min_tokens_per_device"],
              "| T", v["measured"]["tokens_per_device"], "| restore hidden (measured)",
              v["measured"]["restore_hidden_measured"], v["measured"]["fwd_over_half_bwd_gemm"])


if __name__ == "__main__":
    main()
