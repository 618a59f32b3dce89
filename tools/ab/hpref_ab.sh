# SwiGLU' epilogue: L2 prefetch of h (default) vs none (FSEP_H_PREFETCH=0); DRAM of the
# down-dgrad launch and full step (Mixtral, fine), 3 alternations
o=gpurun_out/r02hp; mkdir -p $o
for v in 1 0; do
  for c in mixtral fine; do
    FSEP_H_PREFETCH=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:grouped_gemm_pair --csv --print-units base --log-file $o/dram_${c}_$v.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
    python - $o/dram_${c}_$v.csv <<'PY'
import csv, sys, collections
d = collections.defaultdict(list)
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 14 and r[0] != "ID" and "<0, 1, 0, 2>" in r[4]: d[r[-3]].append(float(r[-1].replace(",", "")))
t, b = d["gpu__time_duration.sum"], d["dram__bytes_read.sum"]
print(sys.argv[1].split("/")[-1], "down-dgrad ms %.3f read GB %.2f" % (sum(t) / len(t) / 1e6, sum(b) / len(b) / 1e9))
PY
  done
done
for rep in 1 2 3; do
  for v in 1 0; do
    FSEP_H_PREFETCH=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
    FSEP_H_PREFETCH=$v python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, statistics
for c in ("mix", "fine"):
    for v in ("1", "0"):
        vals = [json.loads(open(f).read().strip().splitlines()[-1])["value"] for f in sorted(glob.glob(f"gpurun_out/r02hp/{c}_{v}_*.json"))]
        print(c, v, [round(x) for x in vals], round(statistics.mean(vals)))
PY
