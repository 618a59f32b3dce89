# full-step A/B of wave synchronisation per GEMM kind (bit k = GemmKind k: 0 gate-up, 1 down,
# 2 down-dgrad, 3 up-dgrad, 4 wgrad), alternated 3x, Mixtral and fine at N=1
o=gpurun_out/r02ws; mkdir -p $o
for rep in 1 2 3; do
  for kinds in 0x1F 0x0F 0x1B 0x0B; do
    FSEP_WAVE_SYNC_KINDS=$kinds python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${kinds}_$rep.json 2>/dev/null
    FSEP_WAVE_SYNC_KINDS=$kinds python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${kinds}_$rep.json 2>/dev/null
  done
done
