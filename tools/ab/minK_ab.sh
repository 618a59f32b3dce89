# fine config: wave synchronisation for the short-K (K = H = 2048) M-grouped launches too
# (FSEP_WAVE_SYNC_MIN_K=0) vs default (K >= 4096); DRAM per launch and full step, 3 alternations
o=gpurun_out/r02mk; mkdir -p $o
for v in 4096 0; do
  FSEP_WAVE_SYNC_MIN_K=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:grouped_gemm_pair --csv --print-units base --log-file $o/dram_$v.csv python bench.py --config fine --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  python - $o/dram_$v.csv <<'PY'
import csv, sys, collections
d = collections.defaultdict(lambda: collections.defaultdict(list))
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 14 and r[0] != "ID": d[r[4].split("(")[0]][r[-3]].append(float(r[-1].replace(",", "")))
for k, m in d.items():
    t, b = m["gpu__time_duration.sum"], m["dram__bytes_read.sum"]
    print(sys.argv[1].split("/")[-1], k, "ms %.3f" % (sum(t) / len(t) / 1e6), "read GB %.2f" % (sum(b) / len(b) / 1e9))
PY
done
for rep in 1 2 3; do
  for v in 4096 0; do
    FSEP_WAVE_SYNC_MIN_K=$v python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, statistics
for v in ("4096", "0"):
    vals = [json.loads(open(f).read().strip().splitlines()[-1])["value"] for f in sorted(glob.glob(f"gpurun_out/r02mk/fine_{v}_*.json"))]
    print("fine", v, [round(x) for x in vals], round(statistics.mean(vals)))
PY
