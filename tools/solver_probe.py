"""Time the solver loop on a C3-sized slab (64 x 2048^2) and its kernels. GPU only."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28756_b200 as tf  # noqa: E402
from paper_2603_28756_b200.qggmrf import (energy_fid, prior_energy_update, prior_update,  # noqa: E402
                                          stencil_3d)
from paper_2603_28756_b200.toeplitz import FidelityContext  # noqa: E402

z = int(os.environ.get("PROBE_SLICES", "64"))
n = 2048
ang = np.linspace(0, np.pi, 128, endpoint=False)
geom = tf.ScanGeometry(angles=ang, detector_bins=2048, image_side=n)
psf = tf.build_psf(tf.polar_sampling(geom), n)
dev = "cuda"
f = torch.randn((z, n, n), device=dev) * 0.1
fp = f + 0.01 * torch.randn_like(f)
kf, kfp, rs = torch.randn_like(f), torch.randn_like(f), torch.randn_like(f)
out = torch.empty_like(f)
prm = tf.QggmrfParams(sigma=0.5, lam=5e-4)
st = stencil_3d()


def ev(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {}
res["k4_prior_update_ms"] = ev(lambda: prior_update(prm, st, f, fp, out, kf=kf, kfp=kfp, rstar=rs,
                                                    c=0.3, lam=5e-4, inv_L=1e-3))
res["k5_energy_fid_ms"] = ev(lambda: energy_fid(prm, st, out, f=f, kfn=kf, kf=kfp, rstar=rs))
state = torch.tensor([0.0, 0.0, 0.0, 2.0, 0.0], dtype=torch.float64, device=dev)
sums = torch.zeros(4, dtype=torch.float64, device=dev)
res["k45_energy_update_ms"] = ev(lambda: prior_energy_update(
    prm, st, f, fp, out, kf=kf, kfp=kfp, rstar=rs, state=state, lam=5e-4, inv_L=1e-3,
    energy=sums[0], fid=sums[1], dfid=sums[2], gsq=sums[3]))
res["k5_fid_only_ms"] = ev(lambda: energy_fid(prm, st, out, f=f, kfn=kf, kf=kfp, rstar=rs,
                                              with_prior=False))
ctx = FidelityContext(psf=psf, rstar=rs, g_norm_sq=1.0)
cfg = tf.SolverConfig(max_iters=10, tol=1e-300, lipschitz=1e4)
tf.solve(ctx, prm, tf.SolverConfig(max_iters=2, tol=1e-300, lipschitz=1e4), f)
torch.cuda.synchronize()
t0 = time.perf_counter()
_, recs = tf.solve(ctx, prm, cfg, f)
torch.cuda.synchronize()
res["solve_ms_per_iter_wall"] = (time.perf_counter() - t0) / 10 * 1e3
res["step_times_ms"] = [round(r.step_time * 1e3, 3) for r in recs[1:]]
print(json.dumps(res))
