# wgrad tile order: the old default (16-tile m-chunks, FSEP_WGRAD_RASTER=16) vs the adaptive rule (-1 = default:
# n-fastest when a group has no more n tiles than m tiles); DRAM per wgrad launch (ncu) and full step
o=gpurun_out/r02wr2; mkdir -p $o
for v in 16 -1; do
  FSEP_WGRAD_RASTER=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:grouped_gemm_pair --csv --print-units base --log-file $o/dram_$v.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  python - $o/dram_$v.csv <<'PY'
import csv, sys, collections
d = collections.defaultdict(list)
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 14 and r[0] != "ID" and "<1, 1, 1, 3>" in r[4]: d[r[-3]].append(float(r[-1].replace(",", "")))
print(sys.argv[1], [round(x / 1e6, 3) for x in d["gpu__time_duration.sum"]], [round(x / 1e9, 2) for x in d["dram__bytes_read.sum"]])
PY
done
for rep in 1 2 3; do
  for v in 16 -1; do
    FSEP_WGRAD_RASTER=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
    FSEP_WGRAD_RASTER=$v python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob
o = "gpurun_out/r02wr2"
for c in ("mix", "fine"):
    for v in ("16", "-1"):
        vals = []
        for f in sorted(glob.glob(f"{o}/{c}_{v}_*.json")):
            d = json.loads(open(f).read().strip().splitlines()[-1]); vals.append((round(d["value"]), d["phases_ms_layer0"]["bwd_gemms"]))
        print(c, v, vals)
PY
