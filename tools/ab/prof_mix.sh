# Mixtral N=1: bench line, ncu launch list, ncu --set full of one step's kernels
python bench.py --steps 10 --warmup 3 > gpurun_out/r1m.json 2> gpurun_out/r1m.err; echo b=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1_mixtral.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm|dispatch|combine|unpermute|router|plan_kernel|block_scan" -s 40 -c 30 -o gpurun_out/prof_mix python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_f.log 2>&1; echo ncuf=$?
