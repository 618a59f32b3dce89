# NCCL transport (FSEP_COMM=nccl) at N GPUs: real multi-GPU tests, then the step vs the copy engines
o=gpurun_out/r02nc; mkdir -p $o
n=$(nvidia-smi -L | wc -l)
python -m pytest tests/test_gpu_multiprocess.py -q --timeout 900 > $o/mp.log 2>&1; echo mp=$?; tail -3 $o/mp.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29551"
for rep in 1 2; do
  for comm in ce nccl; do
    FSEP_COMM=$comm timeout 900 $R bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-ep --no-local-first --no-static > $o/mix_${comm}_$rep.json 2> $o/mix_${comm}_$rep.err; echo mix $comm=$?
    FSEP_COMM=$comm timeout 900 $R bench.py --config fine --gpus $n --steps 10 --warmup 3 --no-e2e --no-ep --no-local-first --no-static > $o/fine_${comm}_$rep.json 2> $o/fine_${comm}_$rep.err; echo fine $comm=$?
  done
done
