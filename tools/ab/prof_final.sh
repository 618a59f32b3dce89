# N=1 ncu evidence for both configs: launch lists (gpu__time_duration) + --set full of one step,
# summarised on the box (the .ncu-rep files are too large to bring back)
for cfg in mixtral fine; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1_$cfg.csv python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l_$cfg.log 2>&1; echo ncul=$?
timeout 1200 ncu --set full --clock-control none -k regex:"grouped_gemm|dispatch|combine|unpermute|router|plan_kernel|block_scan|expand|grad_rs" -s 40 -c 30 -o /tmp/prof_$cfg python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_f_$cfg.log 2>&1; echo ncuf=$?
python tools/ncu_summary.py /tmp/prof_$cfg.ncu-rep gpurun_out/ncu_full_n1_$cfg.txt --traffic gpurun_out/gemm_traffic_$cfg.json --header "ncu --set full --clock-control none, bench.py --config $cfg N=1 (one step after 3 warm-up steps; -s 40 -c 30)\nround 1 final kernels: wave-synchronised long-K GEMMs, LPT/snake wgrad schedule, cta-scope TMEM release"; echo sum=$?
done
ls -la gpurun_out
