"""e2e fidelity_grad with host float64 buffers (64 x 2048^2), more timed steps than
bench.py, under the current TF_STAGE_THREADS / TF_PIPE_MB.  GPU only."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28756_b200 as tf  # noqa: E402
from paper_2603_28756_b200.radon import back_project_stack  # noqa: E402

ang = np.linspace(0, np.pi, 128, endpoint=False)
geom = tf.ScanGeometry(angles=ang, detector_bins=2048, image_side=2048)
plan = tf.NufftPlan(2048, tf.polar_sampling(geom), 1e-6)
psf = tf.build_psf(plan.sampling, 2048)
g = torch.randn((64, 128, 2048), device="cuda")
ctx = tf.FidelityContext(psf=psf, rstar=back_project_stack(plan, g), g_norm_sq=1.0)
f = np.random.default_rng(5).standard_normal((64, 2048, 2048))
for _ in range(3):
    tf.fidelity_grad(ctx, f)
times = []
for _ in range(8):
    t0 = time.perf_counter()
    out = tf.fidelity_grad(ctx, f)
    _ = float(out[-1, -1, -1])
    del out
    times.append(time.perf_counter() - t0)
times.sort()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("TF_")},
                  "cpus": os.cpu_count(), "median_evals_s": 64 / times[len(times) // 2],
                  "best_evals_s": 64 / times[0], "worst_evals_s": 64 / times[-1]}))
