# full-step A/B of the M-grouped tile raster (m-chunk size), Mixtral N=1, alternated 3x
o=gpurun_out/r02mr; mkdir -p $o
for rep in 1 2 3; do
  for v in 16 8 32 64; do
    FSEP_MRASTER=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${v}_$rep.json 2>/dev/null
  done
done
