python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/gemm_perf.py 2048 1408 64 4096; timeout 300 python tools/gemm_perf.py 4096 14336 8 4096; done
