"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck).  GPU only; sizes kept small so the instrumented run stays short."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28756_b200 as tf  # noqa: E402
from paper_2603_28756_b200.radon import back_project_stack, fbp_stack, forward_project_stack  # noqa: E402

n = int(os.environ.get("SAN_N", "256"))
if os.environ.get("SAN_MODE") == "toeplitz":
    # the Toeplitz chain alone (N = 1024: the two-pass radix-64 column kernel on
    # M = 2048 with its named barriers, mbarriers and TMA), even and odd Nd, 5 slices
    # (uneven over the kernel's four slice groups)
    ang = np.linspace(0, np.pi, 16, endpoint=False)
    for nd in (n, n + 1):
        geom = tf.ScanGeometry(angles=ang, detector_bins=nd, image_side=n)
        psf = tf.build_psf(tf.polar_sampling(geom), n)
        x = torch.randn((5, n, n), device="cuda")
        y = tf.toeplitz_apply(psf, x)
    torch.cuda.synchronize()
    print("sanitize workload done", float(y.abs().sum()))
    sys.exit(0)
ang = np.linspace(0, np.pi, 24, endpoint=False)
geom = tf.ScanGeometry(angles=ang, detector_bins=n, image_side=n)
plan = tf.NufftPlan(n, tf.polar_sampling(geom), 1e-6)
psf = tf.build_psf(plan.sampling, n)
x = torch.randn((3, n, n), device="cuda")
g = torch.randn((3, 24, n), device="cuda")
y = tf.toeplitz_apply(psf, x)
rs = back_project_stack(plan, g)
f0 = fbp_stack(plan, g)
p = forward_project_stack(plan, x)
ctx = tf.FidelityContext(psf=psf, rstar=rs, g_norm_sq=float((g.double() ** 2).sum()))
prm = tf.QggmrfParams(sigma=0.3, lam=0.05)
rec, _ = tf.solve(ctx, prm, tf.SolverConfig(max_iters=3, tol=1e-300, lipschitz=1e4), f0)
up = tf.upsample(torch.randn((2, n // 2, n // 2), device="cuda"), n, 4)
torch.cuda.synchronize()
print("sanitize workload done", float(y.abs().sum()), float(rec.abs().sum()), float(up.abs().sum()))
