# wgrad tile order: default (16-tile m-chunks) vs n-inner (FSEP_WGRAD_RASTER=2), with K-snake and
# wave-synchronised wgrad; DRAM per wgrad launch (ncu) and full step, 3 alternations
o=gpurun_out/r02wr; mkdir -p $o
for v in 0 2; do
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
  for v in 0 2; do
    FSEP_WGRAD_RASTER=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
    FSEP_WGRAD_RASTER=$v python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob
o = "gpurun_out/r02wr"
for c in ("mix", "fine"):
    for v in ("0", "2"):
        vals = []
        for f in sorted(glob.glob(f"{o}/{c}_{v}_*.json")):
            d = json.loads(open(f).read().strip().splitlines()[-1]); vals.append((round(d["value"]), d["phases_ms_layer0"]["bwd_gemms"]))
        print(c, v, vals)
PY
