#!/bin/bash
# A/B of the prior kernels: tools/solver_probe.py per library (default + variants/lib_*.so),
# libraries interleaved; then the solver parity tests on every variant
mkdir -p gpurun_out
out=gpurun_out/k45_ab.txt; : > $out
for rep in 1 2; do
  for lib in paper_2603_28756_b200/libtomoforge_b200.so variants/lib_*.so; do
    echo "$lib $(TF_LIB_PATH=$PWD/$lib timeout 300 python tools/solver_probe.py 2>&1 | tail -1)" >> $out
  done
done
for lib in variants/lib_*.so; do
  echo "== $lib" >> gpurun_out/k45_tests.log
  TF_LIB_PATH=$PWD/$lib timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_configs.py -x -q -k "fused or c1 or solve_matches or prior_kernels" >> gpurun_out/k45_tests.log 2>&1
done
