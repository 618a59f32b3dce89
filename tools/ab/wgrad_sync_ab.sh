# fine config: wave-synchronised wgrad for every group size (FSEP_WAVE_SYNC_WGRAD=all) vs default
o=${O:-gpurun_out/r02ws}; mkdir -p $o
FSEP_WAVE_SYNC_WGRAD=all python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize.py -q -x > $o/pytest.log 2>&1; rc=$?; tail -1 $o/pytest.log; [ $rc -ne 0 ] && exit 1
for v in default all; do
  if [ $v = all ]; then export FSEP_WAVE_SYNC_WGRAD=all; else unset FSEP_WAVE_SYNC_WGRAD; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:grouped_gemm_pair --csv --print-units base --log-file $o/dram_$v.csv python bench.py --config fine --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  python - $o/dram_$v.csv <<'PY'
import csv, sys, collections
d = collections.defaultdict(list)
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 14 and r[0] != "ID" and "<1, 1, 1, 3>" in r[4]: d[r[-3]].append(float(r[-1].replace(",", "")))
print(sys.argv[1], "wgrad launches", len(d["gpu__time_duration.sum"]), "mean ms %.3f" % (sum(d["gpu__time_duration.sum"]) / len(d["gpu__time_duration.sum"]) / 1e6), "mean read GB %.2f" % (sum(d["dram__bytes_read.sum"]) / len(d["dram__bytes_read.sum"]) / 1e9))
PY
done
unset FSEP_WAVE_SYNC_WGRAD
for rep in 1 2 3; do
  for v in default all; do
    if [ $v = all ]; then export FSEP_WAVE_SYNC_WGRAD=all; else unset FSEP_WAVE_SYNC_WGRAD; fi
    python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
    python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
  done
done
unset FSEP_WAVE_SYNC_WGRAD
python - <<'PY'
import json, glob
import os; o = os.environ.get("O", "gpurun_out/r02ws")
for c in ("fine", "mix"):
    for v in ("default", "all"):
        vals = []
        for f in sorted(glob.glob(f"{o}/{c}_{v}_*.json")):
            d = json.loads(open(f).read().strip().splitlines()[-1]); vals.append((round(d["value"]), d["phases_ms_layer0"]["bwd_gemms"]))
        print(c, v, vals)
PY
