# N=4 A/B: TMEM-accumulator release scope (epilogues store rows to peers over NVLink)
python -m pytest tests/test_gpu_multiprocess.py -x -q 2>&1 | tail -1
for cfg in fine mixtral; do for s in cluster cta; do
FSEP_TMEM_RELEASE=$s python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/ab4_${cfg}_$s.json 2> gpurun_out/ab4_${cfg}_$s.err
python tools/show.py gpurun_out/ab4_${cfg}_$s.json 2>&1 | head -2
done; done
