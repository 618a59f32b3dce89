# A/B: TMEM-accumulator release with .cta-scope (default) vs .cluster-scope release semantics
python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q 2>&1 | tail -2
for i in 1 2; do
for s in cluster cta; do
FSEP_TMEM_RELEASE=$s python bench.py --config fine --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_fine_$s$i.json 2>/dev/null
python tools/show.py gpurun_out/ab_fine_$s$i.json 2>&1 | head -2
FSEP_TMEM_RELEASE=$s python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_mix_$s$i.json 2>/dev/null
python tools/show.py gpurun_out/ab_mix_$s$i.json 2>&1 | head -2
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"router_stream" -c 1 -o gpurun_out/prof_router python bench.py --config fine --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu=$?
