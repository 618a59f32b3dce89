# N=4: multi-process parity tests + bench lines (rs_sum phase after the unrolled streaming sum kernel)
python -m pytest tests/test_gpu_multiprocess.py -x -q 2>&1 | tail -1
for cfg in mixtral fine; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/rs4_${cfg}.json 2> gpurun_out/rs4_${cfg}.err
python tools/show.py gpurun_out/rs4_${cfg}.json 2>&1 | grep -E "json|rs_sum|step_total \[" 
done
