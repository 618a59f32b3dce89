import json, sys
for f in sys.argv[1:]:
    txt = [l for l in open(f) if l.startswith("{")]
    if not txt:
        print(f, "no json"); continue
    d = json.loads(txt[-1]); r = d["roofline"]
    print(f, round(d["value"]), round(d["ms_per_step"], 2), r["achieved"], r["step_frac"],
          (d.get("static_ep") or {}).get("speedup_laer_over_static"), d["clocks"]["sm_mhz"])
    print({k: v for k, v in (d.get("phases_ms_layer0") or {}).items() if v > 0.05})
    for k, v in (d.get("phases_ms_per_rank_layer0") or {}).items():
        print("  ", k, v)
    tk = d.get("token_kernels_layer0") or {}
    print("  token kernels:", {k: (v["ms"], v.get("GBps"), v.get("nvlink_GBps", v.get("effective_GBps_per_sending_gpu"))) for k, v in tk.items()})
