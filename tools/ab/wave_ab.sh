# A/B: wave-synchronised producers in the M-grouped pair GEMMs (FSEP_WAVE_SYNC=1)
python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q 2>&1 | tail -1
FSEP_WAVE_SYNC=1 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1
for ws in 1 0; do
FSEP_WAVE_SYNC=$ws ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:grouped_gemm_pair -s 6 -c 6 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu 2>&1 | grep -E "grouped_gemm_pair_kernel<|dram__|duration|per_second" | sed 's/(CUtensorMap_st.*//'
done
for i in 1 2; do for ws in 0 1; do
FSEP_WAVE_SYNC=$ws python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_mix_$ws$i.json 2>/dev/null
python tools/show.py gpurun_out/ab_mix_$ws$i.json 2>&1 | head -2
done; done
