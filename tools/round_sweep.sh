# Round sweep on one 4-GPU box: GPU tests, N=1/2/4 bench lines (Mixtral + fine), 4-layer drifting config at N=4.
# JSON lines land in gpurun_out/sw_*.json
python -m pytest tests -m gpu -x -q > gpurun_out/sw_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/sw_pytest.log
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sw_smoke.log 2>&1; echo smoke=$?
for cfg in mixtral fine; do
CUDA_VISIBLE_DEVICES=0 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/sw_n1_$cfg.json 2> gpurun_out/sw_n1_$cfg.err; echo n1$cfg=$?
done
for N in 2 4; do for cfg in mixtral fine; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N bench.py --gpus $N --config $cfg --steps 10 --warmup 3 > gpurun_out/sw_n${N}_$cfg.json 2> gpurun_out/sw_n${N}_$cfg.err; echo n$N$cfg=$?
done; done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29569 bench.py --gpus 4 --config multilayer --steps 6 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/sw_n4_multilayer.json 2> gpurun_out/sw_n4_multilayer.err; echo ml=$?
CUDA_VISIBLE_DEVICES=0 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/sw_ref_n1.json 2> gpurun_out/sw_ref_n1.err; echo ref=$?
