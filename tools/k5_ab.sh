#!/bin/bash
# radix-5 (C5) apply A/B: parity tests on the default library, then tools/toeplitz_sweep.py
# at 16 x 2560^2 (M = 5120) per library, interleaved
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_toeplitz.py tests/test_gpu_configs.py -x -q -k "2560 or wedge or midsize or c5" > gpurun_out/k5_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/k5_tests.log
out=gpurun_out/k5_ab.txt; : > $out
for rep in 1 2; do
  for lib in paper_2603_28756_b200/libtomoforge_b200.so variants/lib_*.so; do
    echo "$lib $(SWEEP_N=2560 SWEEP_SLICES=${K5_SLICES:-16} TF_LIB_PATH=$PWD/$lib timeout 300 python tools/toeplitz_sweep.py 2>&1 | tail -1)" >> $out
  done
done
