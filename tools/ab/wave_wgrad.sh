# A/B: wave sync also on the Mixtral wgrad GEMMs
python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q 2>&1 | tail -1
FSEP_WAVE_SYNC_WGRAD=1 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"grouped_gemm_pair_kernel<1" -s 2 -c 2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu 2>&1 | grep -E "dram__|duration|per_second"
FSEP_WAVE_SYNC_WGRAD=0 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"grouped_gemm_pair_kernel<1" -s 2 -c 2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu 2>&1 | grep -E "dram__|duration|per_second"
for i in 1 2; do for ws in 0 1; do
FSEP_WAVE_SYNC_WGRAD=$ws python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_mix_$ws$i.json 2>/dev/null
python tools/show.py gpurun_out/ab_mix_$ws$i.json 2>&1 | head -2
done; done
