# N=4 + fine N=1 A/B of the wave-synchronised M-grouped GEMMs
python -m pytest tests/test_gpu_multiprocess.py -x -q 2>&1 | tail -1
for ws in 0 1; do
FSEP_WAVE_SYNC=$ws CUDA_VISIBLE_DEVICES=0 python bench.py --config fine --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_fine_$ws.json 2>/dev/null
python tools/show.py gpurun_out/ab_fine_$ws.json 2>&1 | head -2
done
for cfg in mixtral fine; do for ws in 0 1; do
FSEP_WAVE_SYNC=$ws python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/ab4_${cfg}_$ws.json 2> gpurun_out/ab4_${cfg}_$ws.err
python tools/show.py gpurun_out/ab4_${cfg}_$ws.json 2>&1 | grep -E "json|gemm_ms"
done; done
