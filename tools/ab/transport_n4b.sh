# copy-engine lanes per destination: raw restore probe, then the step at T=4096 / 16384
o=gpurun_out/r02t2; mkdir -p $o
n=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $R tools/transport_probe.py $o/probe_n$n.json > $o/probe.log 2>&1; echo probe=$?
for T in 4096 16384; do
  for k in 1 2; do
    FSEP_CE_STREAMS=$k timeout 900 $R bench.py --gpus $n --steps 10 --warmup 3 --tokens $T --no-e2e --no-ep --no-local-first --no-static > $o/mix_T${T}_k$k.json 2> $o/mix_T${T}_k$k.err; echo mix $T $k=$?
  done
  for k in 1 2; do
    FSEP_CE_STREAMS=$k timeout 900 $R bench.py --config fine --gpus $n --steps 10 --warmup 3 --tokens $((T*2)) --no-e2e --no-ep --no-local-first --no-static > $o/fine_T$((T*2))_k$k.json 2> $o/fine_T$((T*2))_k$k.err; echo fine $T $k=$?
  done
done
