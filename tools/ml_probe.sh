N=${1:-4}
python -m pytest tests/test_gpu_multiprocess.py -x -q -k modes 2>&1 | tail -1
for pf in "" "--no-prefetch" "" "--no-prefetch"; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --config multilayer $pf --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/ml.json 2> gpurun_out/ml.err
grep "^{" gpurun_out/ml.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_rank_layer0']; print('pf=$pf', round(d['value']), round(d['ms_per_step'],2), 'gu', p['fwd_gemm_gateup'], 'gemm', p['gemm_ms'])"
done
