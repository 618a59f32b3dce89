# Mixtral: adaptive wgrad raster (default) vs 16-tile m-chunks, 4 alternations
o=gpurun_out/r02wr3; mkdir -p $o
for rep in 1 2 3 4; do
  for v in 16 -1; do
    FSEP_WGRAD_RASTER=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, statistics
for v in ("16", "-1"):
    vals = [json.loads(open(f).read().strip().splitlines()[-1])["value"] for f in sorted(glob.glob(f"gpurun_out/r02wr3/mix_{v}_*.json"))]
    print(v, [round(x) for x in vals], round(statistics.mean(vals)))
PY
