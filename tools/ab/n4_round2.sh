# N=4 round-2 measurements: multilayer deferred-RS A/B, NVLink counters of the Mixtral step,
# and the configs[4] skew sweep (FSEP vs static EP)
o=gpurun_out/r02n4; mkdir -p $o
n=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541"
for rep in 1 2; do
  timeout 900 $R bench.py --config multilayer --gpus $n --steps 6 --warmup 3 --no-e2e --no-ep --no-local-first --no-static > $o/ml_base_$rep.json 2> $o/ml_base_$rep.err; echo ml base=$?
  timeout 900 $R bench.py --config multilayer --gpus $n --steps 6 --warmup 3 --no-e2e --no-ep --no-local-first --no-static --defer-rs > $o/ml_defer_$rep.json 2> $o/ml_defer_$rep.err; echo ml defer=$?
done
# NVLink bytes: 3 warm-up + 10 timed steps, nothing else
timeout 900 python tools/nvlink_counters.py $o/nvlink_mix.json -- $R bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-ep --no-local-first --no-static --no-cpu > $o/nvl_mix.json 2> $o/nvl_mix.err; echo nvl=$?
timeout 900 python tools/nvlink_counters.py $o/nvlink_fine.json -- $R bench.py --config fine --gpus $n --steps 10 --warmup 3 --no-e2e --no-ep --no-local-first --no-static --no-cpu > $o/nvl_fine.json 2> $o/nvl_fine.err; echo nvlf=$?
nvidia-smi nvlink -gt d > $o/nvlink_raw.txt 2>&1
# full lines (e2e, static EP, pure EP, local-first) for both configs
timeout 1200 $R bench.py --gpus $n --steps 10 --warmup 3 > $o/mix_full.json 2> $o/mix_full.err; echo mixfull=$?
timeout 1200 $R bench.py --config fine --gpus $n --steps 10 --warmup 3 > $o/fine_full.json 2> $o/fine_full.err; echo finefull=$?
bash tools/skew_sweep.sh $n > $o/skew.log 2>&1; echo skew=$?
