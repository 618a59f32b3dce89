# N=4 Mixtral: dispatch CTAs per SM 1 (default) vs 2 / 3 -- the NVLink-bound dispatch phase, 2 alternations
o=gpurun_out/r02dc; mkdir -p $o
for rep in 1 2; do
  for v in 1 2 3; do
    FSEP_DISPATCH_CTAS_PER_SM=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800 + rep)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu --no-ep --no-local-first --no-static > $o/mix_${v}_$rep.json 2> $o/mix_${v}_$rep.err
    FSEP_DISPATCH_CTAS_PER_SM=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29810 + rep)) bench.py --gpus 4 --config fine --steps 10 --warmup 3 --no-e2e --no-cpu --no-ep --no-local-first --no-static > $o/fine_${v}_$rep.json 2> $o/fine_${v}_$rep.err
  done
done
python - <<'PY'
import json, glob
for c in ("mix", "fine"):
    for v in ("1", "2", "3"):
        out = []
        for f in sorted(glob.glob(f"gpurun_out/r02dc/{c}_{v}_*.json")):
            try:
                d = json.loads(open(f).read().strip().splitlines()[-1]); p = d["phases_ms_layer0"]
                out.append((round(d["value"]), p["dispatch"], p.get("dispatch_barrier")))
            except Exception as e:
                out.append(str(e)[:40])
        print(c, v, out)
PY
