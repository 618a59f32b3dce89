python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
for i in 1 2; do echo "== bf16 stage"; ONLY=down_dgrad,down_dgrad_plain PLAIN=1 timeout 300 python tools/gemm_perf.py 2048 1408 64 4096; ONLY=down_dgrad,down_dgrad_plain PLAIN=1 timeout 300 python tools/gemm_perf.py 4096 14336 8 4096; done
rm -f paper_2602_11686_b200/lib/obj/grouped_gemm.cu.o paper_2602_11686_b200/lib/obj/debug_capi.cu.o
FSEP_NVCC_EXTRA="-DFSEP_SWIGLU_BWD_F32_STAGE" python -c "from paper_2602_11686_b200 import build; build.build()" > /dev/null 2>&1 || echo BUILD FAILED
for i in 1 2; do echo "== f32 stage"; ONLY=down_dgrad,down_dgrad_plain PLAIN=1 timeout 300 python tools/gemm_perf.py 2048 1408 64 4096; ONLY=down_dgrad,down_dgrad_plain PLAIN=1 timeout 300 python tools/gemm_perf.py 4096 14336 8 4096; done
