"""Where the non-iteration time of a C4-style solve_hierarchical goes: wraps the
setup phases (sinogram upload, strided rows, NUFFT plan + device tables, PSF, R*g,
FBP, Lipschitz estimate, Lanczos upsample) with synchronised timers.  GPU only.
C4_SIDE (default 1024) sets the volume side; iterations (40, 20, 10)."""
import collections
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28756_b200 as tf  # noqa: E402
from paper_2603_28756_b200 import multires, solver  # noqa: E402
from paper_2603_28756_b200.phantoms import shepp_logan_slab  # noqa: E402
from paper_2603_28756_b200.radon import forward_project_stack  # noqa: E402

n = int(os.environ.get("C4_SIDE", "1024"))
ang = np.linspace(0, np.pi, 128, endpoint=False)
geom = tf.ScanGeometry(angles=ang, detector_bins=n, image_side=n)
plan = tf.NufftPlan(n, tf.polar_sampling(geom), 1e-6)
rows = np.empty((n, 128, n), dtype=np.float32)
for z0 in range(0, n, 64):
    r = forward_project_stack(plan, shepp_logan_slab(n, n, z0, min(n, z0 + 64)))
    r += 0.5 * torch.randn(r.shape, device=r.device)
    rows[z0:z0 + 64] = r.cpu().numpy()
sino = tf.Sinogram(angles=ang, data=rows)
del rows
tf.clear_caches()
torch.cuda.empty_cache()

acc = collections.Counter()
cnt = collections.Counter()


def wrap(mod, name, label=None):
    fn = getattr(mod, name)

    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        acc[label or name] += time.perf_counter() - t0
        cnt[label or name] += 1
        return r
    setattr(mod, name, w)


for name in ("_downsample_rows", "build_psf", "back_project_stack", "fbp_stack",
             "upsample_stack", "NufftPlan", "solve_owned"):
    wrap(multires, name)
wrap(multires._device, "to_device", "to_device (sinogram upload)")
wrap(solver, "estimate_lipschitz")
hier = tf.GridHierarchy(levels=(n // 4, n // 2, n), iters_per_level=(40, 20, 10))
prm = tf.QggmrfParams(sigma=0.1, lam=5e-4)
cfg = tf.SolverConfig(max_iters=1, tol=1e-300)
steps = collections.Counter()
per_iter = collections.defaultdict(list)


def rec(lvl, r):
    steps[lvl] += r.step_time
    per_iter[lvl].append((round(1e3 * r.step_time, 1), int(r.restarted)))


torch.cuda.synchronize()
t0 = time.perf_counter()
est, lrecs = multires.solve_hierarchical_device(sino, hier, prm, cfg, use_fbp_init=True,
                                                 on_record=rec)
torch.cuda.synchronize()
total = time.perf_counter() - t0
print(json.dumps({"side": n, "total_s": total,
                  "phases_s": {k: round(v, 4) for k, v in acc.items()},
                  "calls": dict(cnt),
                  "iteration_step_time_s_per_level": {k: round(v, 4) for k, v in steps.items()},
                  "per_iteration_ms_restarted": {k: v for k, v in per_iter.items()}}))
