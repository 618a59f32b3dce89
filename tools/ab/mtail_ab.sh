# M=128 tail tiles: correctness, then full-step A/B (FSEP_GEMM_MTAIL=0 = masked M=256 tail tiles)
o=gpurun_out/r02mt; mkdir -p $o
python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_gpu_ce_virtual.py -q -x --timeout 900 > $o/pytest.log 2>&1; rc=$?; tail -3 $o/pytest.log; echo tests=$rc
[ $rc -ne 0 ] && exit 1
for rep in 1 2; do
  for v in 1 0; do
    FSEP_GEMM_MTAIL=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
    FSEP_GEMM_MTAIL=$v python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2>/dev/null
  done
done
