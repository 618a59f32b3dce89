for i in 1 2; do timeout 300 python tools/gemm_perf.py 4096 14336 8 4096; timeout 300 python tools/gemm_perf.py 2048 1408 64 4096; done
