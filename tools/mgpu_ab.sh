N=${1:-4}
for r in 1 2; do for v in 1 0; do for cfg in mixtral fine; do
FSEP_RESTORE_SPLIT=$v python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config $cfg --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/ab.json 2> gpurun_out/ab.err
grep "^{" gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_rank_layer0']; print('split=$v $cfg', round(d['value']), round(d['ms_per_step'],2), 'disp', p['dispatch'], 'fwd', p['fwd_gemms'])"
done; done; done
