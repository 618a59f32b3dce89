# K-snake kinds x m-raster, full step, 3 alternations (Mixtral and fine, N=1)
o=gpurun_out/r02ks2; mkdir -p $o
for rep in 1 2 3; do
  for cfg in "0:16" "0x1E:16" "0x1F:16" "0x1E:8"; do
    ks=${cfg%%:*}; mr=${cfg##*:}
    FSEP_KSNAKE=$ks FSEP_MRASTER=$mr python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${ks}_${mr}_$rep.json 2>/dev/null
    FSEP_KSNAKE=$ks FSEP_MRASTER=$mr python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${ks}_${mr}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, statistics
o = "gpurun_out/r02ks2"
for c in ("mix", "fine"):
    for cfg in ("0_16", "0x1E_16", "0x1F_16", "0x1E_8"):
        vals = []
        for f in sorted(glob.glob(f"{o}/{c}_{cfg}_*.json")):
            try:
                vals.append(json.loads(open(f).read().strip().splitlines()[-1])["value"])
            except Exception:
                pass
        print(c, cfg, [round(v) for v in vals], "mean %.0f" % statistics.mean(vals) if vals else "")
PY
