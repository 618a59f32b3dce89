N=${1:-4}
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for v in 1 0; do for cfg in fine mixtral; do
FSEP_DEDUPE=$v python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config $cfg --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/ab.json 2> gpurun_out/ab.err
grep "^{" gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_rank_layer0']; ph=d['phases_ms_layer0']; print('dedupe=$v $cfg', round(d['value']), round(d['ms_per_step'],2), 'disp', p['dispatch'], 'dbar', ph['dispatch_barrier'], 'cbwd', p['combine_bwd_router_wgrad'], 'bar0', ph['bwd_barrier0'])" || tail -3 gpurun_out/ab.err
done; done; done
