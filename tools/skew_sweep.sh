# configs[4]: FSEP (laer) vs static EP under Zipf skew 0.0-1.5 at N GPUs (default 4); one JSON line per (config, alpha)
N=${1:-4}
for cfg in mixtral fine; do for a in 0.0 0.3 0.6 0.9 1.2 1.5; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus $N --config $cfg --alpha $a --steps 8 --warmup 3 --no-e2e --no-ep --no-local-first > gpurun_out/skew_n${N}_${cfg}_$a.json 2> gpurun_out/skew_n${N}_${cfg}_$a.err
echo "$cfg $a $?"
done; done
