# Restore/compute overlap vs tokens per device (validates overlap_min_tokens, cost.cpp:123-143)
N=${1:-4}
for T in 2048 4096 8192; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --tokens $T --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/ov_n${N}_t${T}.json 2> gpurun_out/ov_n${N}_t${T}.err; echo T=$T rc=$?
done
