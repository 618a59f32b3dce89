# profile set for the final kernels (K-snake, router staging): ncu launch lists and one-step ncu --set full captures, summarised ON THE BOX
# captures summarised ON THE BOX (the .ncu-rep files exceed gpurun's 64 MiB copy-back limit)
o=${O:-gpurun_out/r02f2}; mkdir -p $o
for c in mixtral fine; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu > $o/ncul_$c.log 2>&1; echo ncul $c=$?
  python tools/launch_summary.py $o/launches_$c.csv $o/launches_$c.txt "ncu --metrics gpu__time_duration.sum --clock-control none: bench.py --config $c --steps 2 --warmup 3 (5 steps; cold-cache serialised launches)" 5 > /dev/null
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm|dispatch|combine|unpermute|router|plan_kernel|block_scan|expand" -s 40 -c 30 -o /tmp/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > $o/ncuf_$c.log 2>&1; echo ncuf $c=$?
  python tools/ncu_summary.py /tmp/full_$c.ncu-rep $o/ncu_full_$c.txt --traffic $o/gemm_traffic_$c.json --header "ncu --set full --clock-control none, bench.py --config $c N=1 (one step after 3 warm-up steps; -s 40 -c 30)" > $o/ncus_$c.log 2>&1; echo sum $c=$?
  ncu -i /tmp/full_$c.ncu-rep --page details --csv > $o/ncu_details_$c.csv 2>/dev/null
  gzip -f $o/ncu_details_$c.csv
  rm -f /tmp/full_$c.ncu-rep
done
rm -f $o/launches_*.csv
