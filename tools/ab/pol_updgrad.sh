# up-dgrad (Mixtral shape): L2 eviction policy of A / B vs DRAM bytes read and time (ncu, cold)
for pol in 15 5 11 14 10 7 13; do
for r in 0 8; do
echo "POL=$pol RASTER=$r"
POL=$pol RASTER=$r ONLY=up_dgrad ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:grouped -s 3 -c 1 python tools/gemm_perf.py 4096 14336 8 4096 2>&1 | grep -E "dram__|duration|per_second"
done; done
