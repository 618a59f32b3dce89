# 7-stage wgrad with direct fp32 stores (-DFSEP_WGRAD7 variant library) vs default:
# correctness of the variant, then isolated GEMM time and the full step, alternated
o=gpurun_out/r02w7; mkdir -p $o
FSEP_LIB_NAME=libmoeplan_b200_w7.so python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x > $o/pytest.log 2>&1; rc=$?; tail -2 $o/pytest.log; echo tests=$rc
[ $rc -ne 0 ] && exit 1
for rep in 1 2 3; do
  for v in libmoeplan_b200.so libmoeplan_b200_w7.so; do
    echo "== $v mixtral"; FSEP_LIB_NAME=$v timeout 300 python tools/gemm_perf.py 4096 14336 8 4096 2>&1 | grep -E "^wgrad"
    echo "== $v fine"; FSEP_LIB_NAME=$v timeout 300 python tools/gemm_perf.py 2048 1408 64 4096 2>&1 | grep -E "^wgrad"
  done
done
for rep in 1 2 3; do
  for v in libmoeplan_b200.so libmoeplan_b200_w7.so; do
    FSEP_LIB_NAME=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
    FSEP_LIB_NAME=$v python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob
o = "gpurun_out/r02w7"
for c in ("mix", "fine"):
    for v in ("libmoeplan_b200.so", "libmoeplan_b200_w7.so"):
        vals = []
        for f in sorted(glob.glob(f"{o}/{c}_{v}_*.json")):
            try:
                d = json.loads(open(f).read().strip().splitlines()[-1]); vals.append((round(d["value"]), d["phases_ms_layer0"]["bwd_gemms"]))
            except Exception as e:
                vals.append(str(e)[:40])
        print(c, v, vals)
PY
