N=${1:-4}
for v in ce kernel; do
if [ $v = kernel ]; then export FSEP_COMM=kernel; fi
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 --no-static --no-ep > gpurun_out/ab_${v}.json 2> gpurun_out/ab_${v}.err
grep "^{" gpurun_out/ab_${v}.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],2), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2))"
done
