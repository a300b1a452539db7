#!/bin/bash
# K2 candidate check: Toeplitz parity tests on the default library, then the A/B sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_toeplitz.py tests/test_gpu_psf.py tests/test_gpu_nufft.py -x -q > gpurun_out/k2try_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/k2try_pytest.log
bash tools/k2_ab.sh
