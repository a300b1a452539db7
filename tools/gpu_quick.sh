#!/bin/bash
# quick GPU check: selected tests + a bench run without the long legs
TAG=${1:-q}
shift
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q "$@" > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-c4 --no-c5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
