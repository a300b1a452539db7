#!/bin/bash
# A/B the variants in variants/lib_*.so against the default library (toeplitz_sweep
# per library), libraries interleaved so box drift hits all of them alike
mkdir -p gpurun_out
out=gpurun_out/k2_ab.txt; : > $out
for rep in 1 2 3; do
  for lib in paper_2603_28756_b200/libtomoforge_b200.so variants/lib_*.so; do
    echo "$lib $(TF_LIB_PATH=$PWD/$lib timeout 300 python tools/toeplitz_sweep.py 2>&1 | tail -1)" >> $out
  done
done
