"""Profile the 3-level C3 hierarchical solve (host cProfile, top functions). GPU only."""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28756_b200 as tf  # noqa: E402

ang = np.linspace(0, np.pi, 128, endpoint=False)
g = np.random.default_rng(0).standard_normal((64, 128, 2048))
sino = tf.Sinogram(angles=ang, data=g)
prm = tf.QggmrfParams(sigma=0.5, lam=5e-4)
hier = tf.GridHierarchy(levels=(512, 1024, 2048), iters_per_level=(40, 20, 10))
cfg = tf.SolverConfig(max_iters=1, tol=1e-300, lipschitz=None)
tf.solve_hierarchical(sino, hier, prm, cfg, use_fbp_init=True)  # warm
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
tf.solve_hierarchical(sino, hier, prm, cfg, use_fbp_init=True)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
