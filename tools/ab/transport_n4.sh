# N-GPU transport A/B (copy engines vs SM push vs NCCL), then the step with each transport
o=gpurun_out/r02t; mkdir -p $o
n=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $R tools/transport_probe.py $o/probe_n$n.json > $o/probe.log 2>&1; echo probe=$?
for T in 4096 16384; do
  for comm in ce sm; do
    FSEP_COMM=$comm timeout 900 $R bench.py --gpus $n --steps 10 --warmup 3 --tokens $T --no-e2e --no-ep --no-local-first --no-static > $o/mix_T${T}_$comm.json 2> $o/mix_T${T}_$comm.err; echo mix $T $comm=$?
  done
done
