"""Time the Toeplitz gradient (64 x 2048^2) and its three kernels under the current
environment (tuning knobs such as TF_K2 are read by the library).  GPU only."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28756_b200 as tf  # noqa: E402
from paper_2603_28756_b200 import _lib  # noqa: E402
from paper_2603_28756_b200.toeplitz import apply_stack  # noqa: E402

z = int(os.environ.get("SWEEP_SLICES", "64"))
n = int(os.environ.get("SWEEP_N", "2048"))
ang = np.linspace(0, np.pi, 128, endpoint=False)
geom = tf.ScanGeometry(angles=ang, detector_bins=n, image_side=n)
psf = tf.build_psf(tf.polar_sampling(geom), n)
x = torch.randn((z, n, n), device="cuda")
rs = torch.randn((z, n, n), device="cuda")
out = torch.empty_like(x)
for _ in range(5):
    apply_stack(psf, x, out=out, aux=rs, alpha=1.0, beta=-1.0)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
steps = 20
a.record()
for _ in range(steps):
    apply_stack(psf, x, out=out, aux=rs, alpha=1.0, beta=-1.0)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / steps
_lib.timing_enable(True)
for _ in range(steps):
    apply_stack(psf, x, out=out, aux=rs, alpha=1.0, beta=-1.0)
torch.cuda.synchronize()
kt = {k: round(t / c, 4) for k, (t, c) in _lib.timing_collect().items()}
_lib.timing_enable(False)
print(json.dumps({"n": n, "fft_side": psf.fft_side, "env": {k: v for k, v in os.environ.items() if k.startswith("TF_")},
                  "ms_per_step": round(ms, 4), "evals_per_s": round(z / ms * 1e3, 1),
                  "kernel_ms": kt}))
