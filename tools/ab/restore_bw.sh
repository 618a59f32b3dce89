# N=4 bench lines with the shard-restore NVLink entry
for cfg in mixtral fine; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/rb_$cfg.json 2> gpurun_out/rb_$cfg.err
python tools/show.py gpurun_out/rb_$cfg.json 2>&1 | grep -E "json|token kernels"
python -c "import json; d=[json.loads(l) for l in open('gpurun_out/rb_$cfg.json') if l.startswith('{')][0]; print(d['token_kernels_layer0'].get('restore'))"
done
