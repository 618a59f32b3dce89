# end-of-round multi-GPU lines with the final code: N=2 and N=4 full bench lines (Mixtral, fine), multilayer at N=4
o=${O:-gpurun_out/r02fm}; mkdir -p $o
for n in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n"
  timeout 1200 $R bench.py --gpus $n --steps 10 --warmup 3 > $o/mix_n$n.json 2> $o/mix_n$n.err; echo mix $n=$?
  timeout 1200 $R bench.py --config fine --gpus $n --steps 10 --warmup 3 > $o/fine_n$n.json 2> $o/fine_n$n.err; echo fine $n=$?
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29569"
timeout 1200 $R bench.py --config multilayer --gpus 4 --steps 6 --warmup 3 --no-static --no-ep --no-local-first > $o/ml_n4.json 2> $o/ml_n4.err; echo ml=$?
timeout 600 $R bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > $o/ref_n4.json 2> $o/ref_n4.err; echo ref=$?
