for i in 1 2 3; do for v in 1 0; do echo "== ntail $v"; FSEP_GEMM_NTAIL=$v ONLY=down_dgrad,wgrad_w2,down timeout 300 python tools/gemm_perf.py 2048 1408 64 4096; done; done
