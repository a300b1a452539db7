"""e2e fidelity_grad (host float64, 64 x 2048^2) under staging-thread counts and
pipeline chunk sizes set on the library module (tuning probe, GPU only)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28756_b200 as tf  # noqa: E402
from paper_2603_28756_b200 import _device  # noqa: E402
from paper_2603_28756_b200.radon import back_project_stack  # noqa: E402

ang = np.linspace(0, np.pi, 128, endpoint=False)
geom = tf.ScanGeometry(angles=ang, detector_bins=2048, image_side=2048)
plan = tf.NufftPlan(2048, tf.polar_sampling(geom), 1e-6)
psf = tf.build_psf(plan.sampling, 2048)
g = torch.randn((64, 128, 2048), device="cuda")
ctx = tf.FidelityContext(psf=psf, rstar=back_project_stack(plan, g), g_norm_sq=1.0)
f = np.random.default_rng(5).standard_normal((64, 2048, 2048))
res = []
for threads in [int(v) for v in os.environ.get("SW_THREADS", "8,16").split(",")]:
    for mb in [int(v) for v in os.environ.get("SW_MB", "64,128,256").split(",")]:
        _device._STAGE_THREADS = threads
        if _device._stage_pool is not None:
            _device._stage_pool.shutdown()
            _device._stage_pool = None
        _device._PIPE_SLICE_BYTES = mb << 20
        for _ in range(2):
            tf.fidelity_grad(ctx, f)
        times = []
        for _ in range(6):
            t0 = time.perf_counter()
            out = tf.fidelity_grad(ctx, f)
            _ = float(out[-1, -1, -1])
            del out
            times.append(time.perf_counter() - t0)
        times.sort()
        res.append({"threads": threads, "chunk_mb": mb, "median_evals_s": 64 / times[3],
                    "best_evals_s": 64 / times[0]})
        print(json.dumps(res[-1]), flush=True)
