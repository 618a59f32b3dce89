# N=4 fine: wave-synchronised wgrad for every group size vs default, 3 alternations
o=gpurun_out/r02ws4; mkdir -p $o
for rep in 1 2 3; do
  for v in default all; do
    if [ $v = all ]; then export FSEP_WAVE_SYNC_WGRAD=all; else unset FSEP_WAVE_SYNC_WGRAD; fi
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + rep)) bench.py --gpus 4 --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${v}_$rep.json 2> $o/fine_${v}_$rep.err
  done
done
unset FSEP_WAVE_SYNC_WGRAD
python - <<'PY'
import json, glob
o = "gpurun_out/r02ws4"
for v in ("default", "all"):
    vals = []
    for f in sorted(glob.glob(f"{o}/fine_{v}_*.json")):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1]); vals.append((round(d["value"]), d["phases_ms_layer0"]["bwd_gemms"]))
        except Exception as e:
            vals.append(str(e)[:60])
    print("fine N=4", v, vals)
PY
