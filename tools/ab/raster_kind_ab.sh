# per-kind m-raster at the Mixtral shape (8 experts x 4096 rows), alternated
for rep in 1 2; do
  for r in 16 8 4 32; do
    echo "== FSEP_MRASTER_1/3=$r"
    FSEP_MRASTER_1=$r FSEP_MRASTER_3=$r timeout 300 python tools/gemm_perf.py 4096 14336 8 4096 2>&1 | grep -E "^(down|up_dgrad) "
  done
done
