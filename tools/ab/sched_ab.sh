# A/B: K-grouped wgrad tile schedule (snake + longest-first groups) vs round robin
python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q 2>&1 | tail -2
for i in 1 2; do
for s in rr snake; do
FSEP_GEMM_SCHED=$s python bench.py --config fine --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_fine_$s$i.json 2>/dev/null
python tools/show.py gpurun_out/ab_fine_$s$i.json 2>&1 | head -2
FSEP_GEMM_SCHED=$s python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_mix_$s$i.json 2>/dev/null
python tools/show.py gpurun_out/ab_mix_$s$i.json 2>&1 | head -2
done; done
