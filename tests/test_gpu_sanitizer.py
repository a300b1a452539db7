"""compute-sanitizer over every kernel family.

Runs tools/sanitize.py (Toeplitz, NUFFT type 1/2, FBP, forward projection,
qGGMRF update/energy, device solver decision, Lanczos upsampling) under
memcheck, racecheck and synccheck at a small size and requires zero errors.
Determinism of the spreading kernel is covered by
test_gpu_nufft.py::test_back_project_deterministic_and_batched."""

import os
import re
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _sanitizer():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    return exe if os.path.exists(exe) else None


# N = 128 runs the generic kernels; N = 512 the TMA / bulk-copy / 256-bit paths and
# interior K4/K5 tiles; N = 1024 "toeplitz" the radix-64 column kernel (M = 2048), N = 2048
# the M = 4096 chain (K1 mirror pass + bulk block copies, K3 bulk row copies), N = 2560
# the radix-5 column kernel of M = 5120
@pytest.mark.parametrize("tool,n,mode", [("memcheck", 128, ""), ("memcheck", 512, ""),
                                         ("racecheck", 128, ""), ("racecheck", 512, ""),
                                         ("synccheck", 512, ""), ("memcheck", 1024, "toeplitz"),
                                         ("racecheck", 1024, "toeplitz"),
                                         ("synccheck", 1024, "toeplitz"),
                                         ("memcheck", 2048, "toeplitz"),
                                         ("racecheck", 2048, "toeplitz"),
                                         ("synccheck", 2048, "toeplitz"),
                                         ("memcheck", 2560, "toeplitz"),
                                         ("racecheck", 2560, "toeplitz"),
                                         ("synccheck", 2560, "toeplitz")])
def test_kernels_clean_under_sanitizer(tool, n, mode):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _sanitizer()
    if exe is None:
        pytest.skip("compute-sanitizer not found")
    env = dict(os.environ, SAN_N=str(n), SAN_MODE=mode, PYTHONPATH=str(ROOT))
    cmd = [exe, "--tool", tool, "--print-limit", "20", sys.executable,
           str(ROOT / "tools" / "sanitize.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = res.stdout + res.stderr
    assert "sanitize workload done" in out, out[-3000:]
    assert re.search(r"ERROR SUMMARY: 0 errors|0 hazards displayed \(0 errors, 0 warnings\)", out), \
        out[-3000:]
