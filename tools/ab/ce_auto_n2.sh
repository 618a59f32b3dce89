# N=2 Mixtral: automatic copy-engine lanes (2 for 176-MB chunks) vs 1 lane, 3 alternations; tiny bench line
o=gpurun_out/r02ce2; mkdir -p $o
for rep in 1 2 3; do
  for v in auto 1; do
    if [ $v = 1 ]; then export FSEP_CE_STREAMS=1; else unset FSEP_CE_STREAMS; fi
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + rep)) bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu --no-ep --no-local-first --no-static > $o/mix_${v}_$rep.json 2> $o/mix_${v}_$rep.err
  done
done
unset FSEP_CE_STREAMS
CUDA_VISIBLE_DEVICES=0 python bench.py --config tiny --steps 10 --warmup 3 > $o/tiny.json 2> $o/tiny.err
python - <<'PY'
import json, glob, statistics
for v in ("auto", "1"):
    vals = [json.loads(open(f).read().strip().splitlines()[-1])["value"] for f in sorted(glob.glob(f"gpurun_out/r02ce2/mix_{v}_*.json"))]
    print("Mixtral N=2", v, [round(x) for x in vals], round(statistics.mean(vals)))
d = json.loads(open("gpurun_out/r02ce2/tiny.json").read().strip().splitlines()[-1])
print("tiny", round(d["value"]), round(d["e2e"]["value"]), d["config"]["l2"])
PY
