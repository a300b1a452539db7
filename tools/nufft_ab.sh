#!/bin/bash
# A/B of the NUFFT libraries: tools/nufft_probe.py per library, interleaved
mkdir -p gpurun_out
out=gpurun_out/nufft_ab.txt; : > $out
for rep in 1 2; do
  for lib in paper_2603_28756_b200/libtomoforge_b200.so variants/lib_*.so; do
    echo "$lib $(TF_LIB_PATH=$PWD/$lib timeout 300 python tools/nufft_probe.py 2>&1 | tail -1)" >> $out
  done
done
