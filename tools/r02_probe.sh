# round-2 baseline probe (GPU box): bench lines, GEMM shapes with/without the fused
# epilogues, and a source-level ncu capture of the down-dgrad (SwiGLU') GEMM.
o=gpurun_out/r02p; mkdir -p $o
python bench.py --steps 20 --warmup 5 > $o/mix.json 2> $o/mix.err; echo mix=$?
python bench.py --config fine --steps 20 --warmup 5 --no-cpu > $o/fine.json 2> $o/fine.err; echo fine=$?
PLAIN=1 python tools/gemm_perf.py 4096 14336 8 4096 > $o/gemm_mix.txt 2>&1; echo gm=$?
PLAIN=1 python tools/gemm_perf.py 2048 1408 64 4096 > $o/gemm_fine.txt 2>&1; echo gf=$?
ONLY=down_dgrad timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_pair -s 3 -c 1 -o $o/dgrad python tools/gemm_perf.py 4096 14336 8 4096 > $o/ncu_dgrad.log 2>&1; echo ncu=$?
ONLY=down_dgrad_plain PLAIN=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_pair -s 3 -c 1 -o $o/dgrad_plain python tools/gemm_perf.py 4096 14336 8 4096 > $o/ncu_dgrad_plain.log 2>&1; echo ncu2=$?
