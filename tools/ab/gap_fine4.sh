# fine N=4: inter-step gap diagnostics (histogram D2H time, planner callback time)
for i in 1 2; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --config fine --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/gapf.json 2> gpurun_out/gapf.err
python - <<'PY'
import json
d=[json.loads(l) for l in open("gpurun_out/gapf.json") if l.startswith("{")][0]
p=d["phases_ms_layer0"]
print("ms/step", round(d["ms_per_step"],2), {k: p.get(k) for k in ("step_total","gap_between_steps","host_planner_wait","hist_on_host_at","planner_done_at","plan","dispatch")})
PY
done
