# K-snake (odd waves stream K backwards): correctness with it on for every GEMM kind, DRAM
# bytes per GEMM launch (ncu, one step), then full-step A/B, 3 alternations per config
o=gpurun_out/r02ks; mkdir -p $o
FSEP_KSNAKE=0x1F python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x --timeout 900 > $o/pytest.log 2>&1; rc=$?; tail -3 $o/pytest.log; echo tests=$rc
[ $rc -ne 0 ] && exit 1
for v in 0 0x1F; do
  FSEP_KSNAKE=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:grouped_gemm_pair --csv --print-units base --log-file $o/dram_$v.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
done
for rep in 1 2 3; do
  for v in 0 0x1F; do
    FSEP_KSNAKE=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
    FSEP_KSNAKE=$v python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, csv, collections
o = "gpurun_out/r02ks"
for c in ("mix", "fine"):
    for v in ("0", "0x1F"):
        vals = []
        for f in sorted(glob.glob(f"{o}/{c}_{v}_*.json")):
            try:
                d = json.loads(open(f).read().strip().splitlines()[-1])
                vals.append((round(d["value"]), d["roofline"]["frac"], d["phases_ms_layer0"]["fwd_gemm_gateup"], d["phases_ms_layer0"]["fwd_gemm_down"], d["phases_ms_layer0"]["bwd_gemms"]))
            except Exception as e:
                vals.append(str(e))
        print(c, v, vals)
for v in ("0", "0x1F"):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for r in csv.reader(open(f"{o}/dram_{v}.csv")):
        if len(r) > 14 and "grouped_gemm_pair" in r[4]:
            k = r[4].split("(")[0].replace("void ", "")
            m, val = r[-3], float(r[-1].replace(",", ""))
            if m == "gpu__time_duration.sum": agg[k][0] += 1; agg[k][1] += val / 1e6
            if m == "dram__bytes_read.sum": agg[k][2] += val / 1e9
            if m == "dram__bytes_write.sum": agg[k][3] += val / 1e9
    for k, (n, ms, rd, wr) in agg.items():
        print(v, k, n, "ms %.3f read GB %.3f write GB %.3f" % (ms / max(n,1), rd / max(n,1), wr / max(n,1)))
PY
