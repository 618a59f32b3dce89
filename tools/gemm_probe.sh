for pol in 0 5 10 2 8; do for r in 8 16 64; do
echo "== POL=$pol RASTER=$r"
POL=$pol RASTER=$r ONLY=up_dgrad,down timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pair_kernel -s 6 -c 2 --csv python tools/gemm_perf.py 4096 14336 8 4096 2>/dev/null | grep -E "pair_kernel" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | sed 's/"//g'
done; done
