o=gpurun_out/r02s; mkdir -p $o
export FSEP_LIB_NAME=libmoeplan_stall.so STALLS=1 PLAIN=1
python tools/gemm_perf.py 4096 14336 8 4096 > $o/mix.txt 2>&1
python tools/gemm_perf.py 2048 1408 64 4096 > $o/fine.txt 2>&1
FSEP_WAVE_SYNC=0 ONLY=down_dgrad,up_dgrad python tools/gemm_perf.py 4096 14336 8 4096 > $o/mix_nows.txt 2>&1
