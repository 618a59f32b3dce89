# fine config: wave-synchronise only the down-dgrad (+SwiGLU') launch (K = 2048) besides the
# wgrads (FSEP_WAVE_SYNC_MIN_K=0 FSEP_WAVE_SYNC_KINDS=0x14) vs default; DRAM of that launch and
# full step, 4 alternations
o=gpurun_out/r02dd; mkdir -p $o
for v in def dd; do
  if [ $v = dd ]; then export FSEP_WAVE_SYNC_MIN_K=0 FSEP_WAVE_SYNC_KINDS=0x14; else unset FSEP_WAVE_SYNC_MIN_K FSEP_WAVE_SYNC_KINDS; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:grouped_gemm_pair --csv --print-units base --log-file $o/dram_$v.csv python bench.py --config fine --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  python - $o/dram_$v.csv <<'PY'
import csv, sys, collections
d = collections.defaultdict(list)
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 14 and r[0] != "ID" and "<0, 1, 0, 2>" in r[4]: d[r[-3]].append(float(r[-1].replace(",", "")))
t, b = d["gpu__time_duration.sum"], d["dram__bytes_read.sum"]
print(sys.argv[1].split("/")[-1], "down-dgrad ms %.3f read GB %.2f" % (sum(t) / len(t) / 1e6, sum(b) / len(b) / 1e9))
PY
done
unset FSEP_WAVE_SYNC_MIN_K FSEP_WAVE_SYNC_KINDS
for rep in 1 2 3 4; do
  for v in def dd; do
    if [ $v = dd ]; then export FSEP_WAVE_SYNC_MIN_K=0 FSEP_WAVE_SYNC_KINDS=0x14; else unset FSEP_WAVE_SYNC_MIN_K FSEP_WAVE_SYNC_KINDS; fi
    python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
unset FSEP_WAVE_SYNC_MIN_K FSEP_WAVE_SYNC_KINDS
python - <<'PY'
import json, glob, statistics
for v in ("def", "dd"):
    vals = [json.loads(open(f).read().strip().splitlines()[-1])["value"] for f in sorted(glob.glob(f"gpurun_out/r02dd/fine_{v}_*.json"))]
    print("fine", v, [round(x) for x in vals], round(statistics.mean(vals)))
PY
