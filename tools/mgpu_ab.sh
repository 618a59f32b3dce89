N=4
python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q 2>&1 | tail -1
run() {
for i in 1 2; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config fine --steps 10 --warmup 3 --no-e2e --no-static --no-ep --no-local-first > gpurun_out/ab.json 2> gpurun_out/ab.err
grep "^{" gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_rank_layer0']; print('$1', round(d['value']), round(d['ms_per_step'],2), 'down', p['fwd_gemm_down'], 'bwd', p['bwd_gemms'])"
done
ONLY=down,up_dgrad timeout 300 python tools/gemm_perf.py 4096 14336 8 4096 | sed "s/ sm .*//" | grep -v total
}
run row128
rm -f paper_2602_11686_b200/lib/obj/grouped_gemm.cu.o paper_2602_11686_b200/lib/obj/debug_capi.cu.o
FSEP_NVCC_EXTRA="-DFSEP_EPI_ROW64" python -c "from paper_2602_11686_b200 import build; build.build()" > /dev/null 2>&1 || echo BUILD FAILED
run row64
