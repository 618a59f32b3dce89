# SwiGLU / SwiGLU' epilogue sigmoid: ex2+rcp (default) vs tanh.approx (-DFSEP_SIGMOID_TANH variant library)
o=gpurun_out/r02sg; mkdir -p $o
FSEP_LIB_NAME=libmoeplan_tanh.so FSEP_NVCC_EXTRA=-DFSEP_SIGMOID_TANH python -c "from paper_2602_11686_b200 import build; build.build()" > $o/build.log 2>&1; echo build=$?
FSEP_LIB_NAME=libmoeplan_tanh.so python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize.py -q -s --timeout 600 > $o/pytest_tanh.log 2>&1; echo tests=$?; grep "full-size" $o/pytest_tanh.log
for rep in 1 2 3; do
  for lib in libmoeplan_b200.so libmoeplan_tanh.so; do
    FSEP_LIB_NAME=$lib python bench.py --config fine --steps 20 --warmup 5 --no-e2e --no-cpu > $o/fine_${lib}_$rep.json 2>/dev/null
    FSEP_LIB_NAME=$lib python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $o/mix_${lib}_$rep.json 2>/dev/null
  done
done
