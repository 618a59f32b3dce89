python -m pytest tests/test_gpu_multiprocess.py -x -q 2>&1 | tail -1
for N in 2 4; do for cfg in mixtral fine; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --config $cfg --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/ab.json 2> gpurun_out/ab.err
grep "^{" gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_rank_layer0']; print('N=$N $cfg', round(d['value']), round(d['ms_per_step'],2), 'rs', p['rs_sum_barrier'], 'bwd', p['bwd_gemms'])"
done; done
