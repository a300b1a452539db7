#!/bin/bash
# A/B sweep of variants/lib_*.so plus one ncu --set full capture of the named K2 kernel
K=${1:-k_cols_conv64}
mkdir -p gpurun_out
bash tools/k2_ab.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
  -o gpurun_out/prof_$K -f python tools/toeplitz_sweep.py > gpurun_out/prof_$K.log 2>&1
