# Mixtral: up-dgrad m-chunk 8 (FSEP_MRASTER_3=8) vs 16 (default), full step, 4 alternations
o=gpurun_out/r02ur; mkdir -p $o
for rep in 1 2 3 4; do
  for v in 16 8; do
    FSEP_MRASTER_3=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, statistics
for v in ("16", "8"):
    vals = [json.loads(open(f).read().strip().splitlines()[-1])["value"] for f in sorted(glob.glob(f"gpurun_out/r02ur/mix_{v}_*.json"))]
    print(v, [round(x) for x in vals], round(statistics.mean(vals)))
PY
