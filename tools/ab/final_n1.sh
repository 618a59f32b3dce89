# HEAD check: N=1 bench lines for both configs + smoke
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in mixtral fine; do
timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/final_n1_$cfg.json 2> gpurun_out/final_n1_$cfg.err
python tools/show.py gpurun_out/final_n1_$cfg.json 2>&1 | head -2
done
