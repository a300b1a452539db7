"""Repeat a 2048^2 apply many times against the oracle to catch async races."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
import oracle as O
import paper_2603_28756_b200 as tf
ang = np.linspace(0, np.pi, 16, endpoint=False)
n = 2048
x = np.random.default_rng(0).standard_normal((3, n, n))
ref = O.apply_batch(O.build_psf(ang, n, n), x)
geom = tf.ScanGeometry(angles=ang, detector_bins=n, image_side=n)
psf = tf.build_psf(tf.polar_sampling(geom), n)
worst = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    out = tf.toeplitz_apply(psf, x)
    err = max(float(np.linalg.norm(out[i] - ref[i]) / np.linalg.norm(ref[i])) for i in range(3))
    worst = max(worst, err)
print('race check: worst rel err over reps:', worst)
