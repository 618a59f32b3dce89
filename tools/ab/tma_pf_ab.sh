# TMA L2 prefetch distance for the pair kernel's operands (FSEP_TMA_PF): correctness with it
# on, isolated GEMM time and full step, Mixtral and fine N=1, 3 alternations
o=gpurun_out/r02pf; mkdir -p $o
FSEP_TMA_PF=6 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x > $o/pytest.log 2>&1; rc=$?; tail -1 $o/pytest.log; [ $rc -ne 0 ] && exit 1
for v in 0 3 6 10; do
  echo "== PF $v"; FSEP_TMA_PF=$v timeout 300 python tools/gemm_perf.py 4096 14336 8 4096 2>&1 | grep -E "^(gateup|down|down_dgrad|up_dgrad|wgrad_w2|wgrad_w13|total)"
done
for rep in 1 2 3; do
  for v in 0 3 6; do
    FSEP_TMA_PF=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
    FSEP_TMA_PF=$v python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, statistics
for c in ("mix", "fine"):
    for v in ("0", "3", "6"):
        vals = [json.loads(open(f).read().strip().splitlines()[-1])["value"] for f in sorted(glob.glob(f"gpurun_out/r02pf/{c}_{v}_*.json"))]
        print(c, v, [round(x) for x in vals], round(statistics.mean(vals)) if vals else None)
PY
