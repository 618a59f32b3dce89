# N=4 Mixtral: where does the time between steps go (device gap, layout H2D, host planner wait)
for lay in laer static; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --steps 10 --warmup 3 --layout $lay --no-e2e --no-static --no-ep --no-local-first > gpurun_out/gap4_$lay.json 2> gpurun_out/gap4_$lay.err
python - $lay <<'PY'
import json,sys
d=[json.loads(l) for l in open(f"gpurun_out/gap4_{sys.argv[1]}.json") if l.startswith("{")][0]
p=d["phases_ms_layer0"]
print(sys.argv[1], "ms/step", round(d["ms_per_step"],2), "step_total", p["step_total"], "layout_h2d", p.get("layout_h2d"), "gap", p.get("gap_between_steps"), "host_wait", p.get("host_planner_wait"))
PY
done
