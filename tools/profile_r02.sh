#!/bin/bash
# Targeted ncu evidence (one GPU): launch list of the default bench step, one full
# capture per hot kernel from the probe scripts, CSV exports (raw / source).
TAG=${1:-r02}
mkdir -p gpurun_out
F="--set full --clock-control none --import-source on"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --no-e2e --no-mbir --no-c4 --no-c5 > /dev/null 2>&1
# Toeplitz step (64 x 2048^2): skip the PSF build and warm-up applies, capture K1, K2, K3
SWEEP_SLICES=64 timeout 900 ncu $F -k regex:'k_rows_fwd_pf|k_cols_conv64|k_rows_inv' -s 12 -c 3 \
  -o gpurun_out/prof_toeplitz_$TAG -f python tools/toeplitz_sweep.py > /dev/null 2>&1
# radix-5 side (16 x 2560^2)
SWEEP_N=2560 SWEEP_SLICES=16 timeout 900 ncu $F -k regex:'k5_rows|k5_cols_conv' -s 12 -c 3 \
  -o gpurun_out/prof_toeplitz5_$TAG -f python tools/toeplitz_sweep.py > /dev/null 2>&1
# solver kernels (64 x 2048^2)
timeout 900 ncu $F -k regex:'k_prior_update_sym|k_energy_fid_t' -s 1 -c 2 \
  -o gpurun_out/prof_solver_$TAG -f python tools/solver_probe.py > /dev/null 2>&1
timeout 900 ncu $F -k regex:'k_prior_energy_update' -s 1 -c 1 \
  -o gpurun_out/prof_k45_$TAG -f python tools/solver_probe.py > /dev/null 2>&1
# one-time kernels (8 x 2048^2)
PROBE_SLICES=8 timeout 900 ncu $F -k regex:'k_spread|k_nufft_rows|k_nufft_cols|k_detector_rows|k_upsample3' \
  -c 6 -o gpurun_out/prof_onetime_$TAG -f python tools/nufft_probe.py > /dev/null 2>&1
timeout 300 python tools/nufft_probe.py > gpurun_out/nufft_probe_$TAG.json 2>&1
timeout 300 python tools/solver_probe.py > gpurun_out/solver_probe_$TAG.json 2>&1
for r in gpurun_out/prof_*_$TAG.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.source.csv 2>/dev/null
  gzip -f $b.source.csv
  rm -f $r
done
ls -la gpurun_out
