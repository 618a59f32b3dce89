# N=4 Mixtral: automatic copy-engine lanes (2 for 88-MB chunks) vs 1 lane, T=16384 and 4096,
# 3 alternations; the multi-process and virtual copy-engine tests first
o=gpurun_out/r02ce; mkdir -p $o
python -m pytest tests/test_gpu_multiprocess.py tests/test_gpu_ce_virtual.py -q -x > $o/pytest.log 2>&1; rc=$?; tail -1 $o/pytest.log; [ $rc -ne 0 ] && exit 1
for rep in 1 2 3; do
  for T in 16384 4096; do
    for v in auto 1; do
      if [ $v = 1 ]; then export FSEP_CE_STREAMS=1; else unset FSEP_CE_STREAMS; fi
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + rep)) bench.py --gpus 4 --tokens $T --steps 20 --warmup 5 --no-e2e --no-cpu --no-ep --no-local-first --no-static > $o/mix_T${T}_${v}_$rep.json 2> $o/mix_T${T}_${v}_$rep.err
    done
  done
done
unset FSEP_CE_STREAMS
python - <<'PY'
import json, glob, statistics
for T in (16384, 4096):
    for v in ("auto", "1"):
        vals = []
        for f in sorted(glob.glob(f"gpurun_out/r02ce/mix_T{T}_{v}_*.json")):
            try: vals.append(json.loads(open(f).read().strip().splitlines()[-1])["value"])
            except Exception as e: pass
        print("Mixtral N=4 T", T, v, [round(x) for x in vals], round(statistics.mean(vals)) if vals else None)
PY
