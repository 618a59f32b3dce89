# weak scaling on one 4-GPU box: N=1 (GPU 0), N=2, N=4, Mixtral and fine, alternated twice
o=${O:-gpurun_out/r02sc}; mkdir -p $o
for rep in 1 2; do
  for cfg in mixtral fine; do
    CUDA_VISIBLE_DEVICES=0 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu > $o/${cfg}_n1_$rep.json 2>/dev/null
    for n in 2 4; do
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --config $cfg --gpus $n --steps 10 --warmup 3 --no-e2e --no-ep --no-local-first --no-static > $o/${cfg}_n${n}_$rep.json 2>/dev/null
    done
  done
done
