"""cProfile of a C4-style solve_hierarchical_device (host-side time by function).
C4_SIDE (default 2048).  GPU only."""
import cProfile
import io
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28756_b200 as tf  # noqa: E402
from paper_2603_28756_b200 import multires  # noqa: E402
from paper_2603_28756_b200.phantoms import shepp_logan_slab  # noqa: E402
from paper_2603_28756_b200.radon import forward_project_stack  # noqa: E402

n = int(os.environ.get("C4_SIDE", "2048"))
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
hier = tf.GridHierarchy(levels=(n // 4, n // 2, n), iters_per_level=(40, 20, 10))
prm = tf.QggmrfParams(sigma=0.1, lam=5e-4)
cfg = tf.SolverConfig(max_iters=1, tol=1e-300)
pr = cProfile.Profile()
torch.cuda.synchronize()
t0 = time.perf_counter()
pr.enable()
est, lrecs = multires.solve_hierarchical_device(sino, hier, prm, cfg, use_fbp_init=True)
torch.cuda.synchronize()
pr.disable()
print("total", time.perf_counter() - t0)
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(40)
print(s.getvalue())
