#!/bin/bash
# One gpurun call: GPU tests, then bench (incl. C4) -- usage: bash tools/gpu_round.sh TAG [pytest-args]
TAG=${1:-r02}
shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rA "$@" > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
