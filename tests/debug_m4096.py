import sys, numpy as np
sys.path.insert(0, '/root/repo')
import oracle as O
import paper_2603_28756_b200 as tf
ang = np.linspace(0, np.pi, 16, endpoint=False)
for n, z in [(2048, 3)]:
    nd = n
    x = np.random.default_rng(0).standard_normal((z, n, n))
    ref = O.apply_batch(O.build_psf(ang, nd, n), x)
    geom = tf.ScanGeometry(angles=ang, detector_bins=nd, image_side=n)
    psf = tf.build_psf(tf.polar_sampling(geom), n)
    out = tf.toeplitz_apply(psf, x)
    d = out[0] - ref[0]
    D = np.abs(np.fft.rfft(np.pad(d, ((0, 0), (0, 2048))), axis=1)).sum(0)
    R = np.abs(np.fft.rfft(np.pad(ref[0], ((0, 0), (0, 2048))), axis=1)).sum(0)
    idx = np.argsort(-D)[:12]
    print('top ky of error:', idx, D[idx] / R[idx])
    # error along x (rows)
    rowerr = np.linalg.norm(d, axis=1) / np.linalg.norm(ref[0], axis=1)
    print('rows with err>1e-3:', np.nonzero(rowerr > 1e-3)[0][:40], len(np.nonzero(rowerr > 1e-3)[0]))
    print('max row err', rowerr.max())
