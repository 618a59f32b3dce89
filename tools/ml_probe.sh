N=${1:-4}
for T in 16384 4096; do for pf in "" "--no-prefetch"; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --config multilayer --tokens $T $pf --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/ml_t${T}${pf}.json 2> gpurun_out/ml_t${T}${pf}.err; echo T=$T pf=$pf rc=$?
grep "^{" gpurun_out/ml_t${T}${pf}.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],2), d['phases_ms_per_rank_layer0']['gemm_ms'])"
done; done
