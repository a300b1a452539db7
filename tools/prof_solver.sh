#!/bin/bash
# solver probe timings + ncu full captures of K45 and K4 (64 x 2048^2)
TAG=${1:-s}
mkdir -p gpurun_out
timeout 300 python tools/solver_probe.py > gpurun_out/solver_probe_$TAG.json 2> gpurun_out/solver_probe_$TAG.err
bash tools/kprof.sh k_prior_energy_update k45_$TAG tools/solver_probe.py
bash tools/kprof.sh k_prior_update_sym k4_$TAG tools/solver_probe.py
python tools/summarize_ncu.py gpurun_out/k45_$TAG.raw.csv gpurun_out/k4_$TAG.raw.csv > gpurun_out/ncu_solver_$TAG.txt 2>&1
