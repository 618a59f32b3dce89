# NVLink bytes per kernel from ncu counters (single-process 2-GPU probe; see tools/nvlink_ncu_probe.py)
o=gpurun_out/r02nv; mkdir -p $o
for c in mixtral fine; do
  timeout 300 python tools/nvlink_ncu_probe.py $c 2 3 > $o/plain_$c.log 2>&1; echo plain $c=$?; tail -1 $o/plain_$c.log
  FSEP_SPIN_TIMEOUT_MS=200 timeout 900 ncu --devices 0 --csv --metrics nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum -k regex:"dispatch_tma|combine_bwd|grouped_gemm_pair|expand_rows|block_scan" --log-file $o/ncu_$c.csv python tools/nvlink_ncu_probe.py $c 2 3 > $o/ncu_$c.log 2>&1; echo ncu $c=$?; tail -1 $o/ncu_$c.log
done
