python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
for i in 1 2; do for cfg in "4096 14336 8 4096" "2048 1408 64 4096"; do
  echo "== $cfg"; PLAIN=1 timeout 300 python tools/gemm_perf.py $cfg
done; done
