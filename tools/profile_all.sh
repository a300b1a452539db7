#!/bin/bash
# ncu evidence for every kernel family (one GPU): launch list of the bench, full
# captures of the Toeplitz, solver and one-time (NUFFT / Lanczos) kernels.
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-mbir > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_rows|k_cols_conv' -s 6 -c 3 \
  -o gpurun_out/prof_toeplitz_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-mbir > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_prior|k_energy' -c 4 \
  -o gpurun_out/prof_solver_$TAG -f python tools/solver_probe.py > /dev/null 2>&1
PROBE_SLICES=8 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'k_spread|k_nufft|k_detector|k_resample|k_upsample|k_plan' -c 14 \
  -o gpurun_out/prof_onetime_$TAG -f python tools/nufft_probe.py > /dev/null 2>&1
timeout 300 python tools/nufft_probe.py > gpurun_out/nufft_probe_$TAG.json 2>&1
timeout 300 python tools/solver_probe.py > gpurun_out/solver_probe_$TAG.json 2>&1

# export the reports to CSV on the box (raw .ncu-rep files exceed gpurun's 64 MiB return cap)
for r in gpurun_out/prof_*_$TAG.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.source.csv 2>/dev/null
  gzip -f $b.source.csv
  rm -f $r
done

ls -la gpurun_out
