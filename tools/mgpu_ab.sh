N=${1:-4}
for v in tma simt tma simt; do
FSEP_DISPATCH=$v python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-static > gpurun_out/ab_${v}.json 2> gpurun_out/ab_${v}.err; python tools/show.py gpurun_out/ab_${v}.json | head -4
done
