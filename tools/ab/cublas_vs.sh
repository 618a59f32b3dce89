# ours (6 grouped launches) vs cuBLAS per-expert matmuls, same box, uniform rows per expert; alternated twice
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
for i in 1 2; do
for shape in "4096 14336 8 4096" "2048 1408 64 4096"; do
echo "== ours $shape"; timeout 300 python tools/gemm_perf.py $shape 2>&1 | tail -7
echo "== cublas $shape"; timeout 300 python tools/cublas_compare.py $shape 2>&1 | tail -7
done; done
