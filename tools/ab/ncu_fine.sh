# ncu --set full of the fine config's SwiGLU-bwd GEMM, down GEMM and router (one launch each)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm_pair_kernel|router_gemm" -s 20 -c 9 -o gpurun_out/prof_fine python bench.py --config fine --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_fine_full.log 2>&1; echo ncuf=$?
