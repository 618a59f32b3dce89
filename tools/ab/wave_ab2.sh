# wave synchronisation on/off, interleaved in one process, cycles per call (tools/gemm_ab.py)
o=gpurun_out/r02w; mkdir -p $o
for gm in down_dgrad up_dgrad down wgrad_w13 wgrad_w2; do
  python tools/gemm_ab.py 4096 14336 8 4096 $gm base=0 nows=0x800 >> $o/mix.txt 2>&1
done
for gm in down_dgrad up_dgrad; do
  python tools/gemm_ab.py 2048 1408 64 4096 $gm base=0 nows=0x800 >> $o/fine.txt 2>&1
done
