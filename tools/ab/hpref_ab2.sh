# h prefetch on (1) / off (0): 4 more alternations, Mixtral and fine
o=gpurun_out/r02hp2; mkdir -p $o
for rep in 1 2 3 4; do
  for v in 1 0; do
    FSEP_H_PREFETCH=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
    FSEP_H_PREFETCH=$v python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, statistics
for c in ("mix", "fine"):
    for v in ("1", "0"):
        vals = [json.loads(open(f).read().strip().splitlines()[-1])["value"] for f in sorted(glob.glob(f"gpurun_out/r02hp2/{c}_{v}_*.json"))]
        print(c, v, [round(x) for x in vals], round(statistics.mean(vals)))
PY
