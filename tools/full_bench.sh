# Round bench sweep: N=1,2,4 for the Mixtral and fine configs (one JSON line each under gpurun_out/)
python bench.py --steps 10 --warmup 3 > gpurun_out/fb_n1_mixtral.json 2> gpurun_out/fb_n1_mixtral.err; echo n1m=$?
python bench.py --config fine --steps 10 --warmup 3 > gpurun_out/fb_n1_fine.json 2> gpurun_out/fb_n1_fine.err; echo n1f=$?
for N in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/fb_n${N}_mixtral.json 2> gpurun_out/fb_n${N}_mixtral.err; echo n${N}m=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --config fine --steps 10 --warmup 3 > gpurun_out/fb_n${N}_fine.json 2> gpurun_out/fb_n${N}_fine.err; echo n${N}f=$?
done
