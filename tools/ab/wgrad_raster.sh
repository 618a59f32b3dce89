# wgrad tile order: longer side outermost (default) vs m-chunks of 16 for both wgrad launches
python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q 2>&1 | tail -1
for i in 1 2; do for r in 16 auto; do
if [ $r = auto ]; then R=; else R=$r; fi
FSEP_WGRAD_RASTER=$R python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_mix_$r$i.json 2>/dev/null
python tools/show.py gpurun_out/ab_mix_$r$i.json 2>&1 | head -2
FSEP_WGRAD_RASTER=$R python bench.py --config fine --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_fine_$r$i.json 2>/dev/null
python tools/show.py gpurun_out/ab_fine_$r$i.json 2>&1 | head -2
done; done
