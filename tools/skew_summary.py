"""Collect the skew sweep (tools/skew_sweep.sh) into one JSON file + a markdown table (dev tool).

  python tools/skew_summary.py gpurun_out 4 profiles/r01_s2_skew_sweep_n4.json
"""
import glob
import json
import sys

src, N, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows = []
for f in sorted(glob.glob(f"{src}/skew_n{N}_*.json")):
    cfg, alpha = f.rsplit("/", 1)[1][len(f"skew_n{N}_"):-5].split("_")
    line = next((l for l in open(f) if l.startswith("{")), None)
    if line is None:
        rows.append({"config": cfg, "alpha": float(alpha), "error": "no JSON line"})
        continue
    d = json.loads(line)
    st = d.get("static_ep") or {}
    rows.append({"config": cfg, "alpha": float(alpha), "laer_tokens_per_s": round(d["value"]),
                 "laer_ms_per_step": round(d["ms_per_step"], 3), "static_ep_tokens_per_s": round(st.get("value", 0)),
                 "static_ep_ms_per_step": round(st.get("ms_per_step", 0), 3),
                 "speedup_laer_over_static": st.get("speedup_laer_over_static"),
                 "step_frac": d["roofline"].get("step_frac"), "clocks": d.get("clocks")})
rows.sort(key=lambda r: (r["config"], r["alpha"]))
json.dump({"n_gpus": N, "command": f"tools/skew_sweep.sh {N}", "rows": rows}, open(out, "w"), indent=1)
print("| config | Zipf α | FSEP (laer) tokens/s | static EP tokens/s | laer ÷ static | step_frac |")
print("|---|---|---|---|---|---|")
for r in rows:
    if "error" in r:
        print(f"| {r['config']} | {r['alpha']} | — | — | — | — |")
        continue
    print(f"| {r['config']} | {r['alpha']} | {r['laer_tokens_per_s']:,} | {r['static_ep_tokens_per_s']:,} | "
          f"{r['speedup_laer_over_static']} | {r['step_frac']} |")
