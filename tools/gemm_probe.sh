python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
for i in 1 2; do ONLY=wgrad_w2,wgrad_w13,up_dgrad timeout 300 python tools/gemm_perf.py 4096 14336 8 4096; ONLY=wgrad_w2,wgrad_w13,up_dgrad timeout 300 python tools/gemm_perf.py 2048 1408 64 4096; done
