# 4 epilogue warps (-DFSEP_EPI_WARPS=4 variant library; no M=128 tail tiles there) vs 8 (default):
# correctness, then full step Mixtral / fine, 3 alternations
o=${O:-gpurun_out/r02e4}; mkdir -p $o
FSEP_LIB_NAME=libmoeplan_b200_e4.so python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_gpu_random_shapes.py tests/test_gpu_shapes.py -q -x > $o/pytest.log 2>&1; rc=$?; tail -1 $o/pytest.log; [ $rc -ne 0 ] && exit 1
for rep in 1 2 3; do
  for v in libmoeplan_b200.so libmoeplan_b200_e4.so; do
    FSEP_LIB_NAME=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
    FSEP_LIB_NAME=$v python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, statistics
for c in ("mix", "fine"):
    for v in ("libmoeplan_b200.so", "libmoeplan_b200_e4.so"):
        vals = [json.loads(open(f).read().strip().splitlines()[-1])["value"] for f in sorted(glob.glob(f"{__import__('os').environ.get('O', 'gpurun_out/r02e4')}/{c}_{v}_*.json"))]
        print(c, v, [round(x) for x in vals], round(statistics.mean(vals)) if vals else None)
PY
