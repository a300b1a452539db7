"""CUDA Lanczos upsampler and the GPU coarse-to-fine driver vs reference fixtures."""

import numpy as np
import pytest

from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_28756_b200 as m

    return m


def test_upsample_matches_reference(tf):
    d = golden("multires.npz")
    assert rel_l2(tf.upsample(d["v"], 20, 6), d["up3"]) < 1e-6
    assert rel_l2(tf.upsample(d["v"][0], 25), d["up2"]) < 1e-6
    g = tf.upsample(tf.ImageGrid(d["v"][0]), 25)
    assert isinstance(g, tf.ImageGrid) and rel_l2(g.data, d["up2"]) < 1e-6


def test_upsample_identity_and_constants(tf):
    """test_multires.py:99-119"""
    x = np.random.default_rng(1).standard_normal((4, 16, 16))
    np.testing.assert_allclose(tf.upsample(x, 16, 4), x, rtol=0, atol=1e-6)
    c = tf.upsample(np.full((3, 8, 8), 2.5), 32, 6)
    np.testing.assert_allclose(c, 2.5, rtol=1e-6)


def test_upsample_c3_level_vs_oracle(tf):
    """(Z/2, 1024^2) -> (Z, 2048^2), the C3 level transfer, on a 4-slice slab."""
    import oracle as O

    x = np.random.default_rng(2).standard_normal((2, 1024, 1024))
    ref = O.upsample(x, 2048, 4)
    assert rel_l2(tf.upsample(x, 2048, 4), ref) < 1e-6


def test_solve_hierarchical_matches_reference(tf):
    d = golden("hier.npz")
    sino = tf.Sinogram(angles=d["angles"], data=d["g"])
    prm = tf.QggmrfParams(sigma=0.1, lam=1e-2)
    hier = tf.GridHierarchy(levels=(16, 32), iters_per_level=(6, 4))
    seen = []
    est, lrecs = tf.solve_hierarchical(sino, hier, prm, tf.SolverConfig(max_iters=1, tol=1e-300),
                                       use_fbp_init=True, on_record=lambda l, r: seen.append(l))
    assert isinstance(est, tf.Volume)
    assert rel_l2(est.data, d["recon"]) < 1e-3
    np.testing.assert_allclose([r.objective for r in lrecs[0]], d["obj0"], rtol=1e-4)
    np.testing.assert_allclose([r.objective for r in lrecs[1]], d["obj1"], rtol=1e-4)
    assert seen == [0] * 7 + [1] * 5


def test_single_level_equals_plain_solve(tf):
    """test_multires.py:168-179: one level == fidelity_context + solve."""
    import torch

    d = golden("solve_3d.npz")
    n = d["f0"].shape[1]
    sino = tf.Sinogram(angles=d["angles"], data=d["g"])
    prm = tf.QggmrfParams(sigma=float(d["sigma"]), lam=float(d["lam"]))
    cfg = tf.SolverConfig(max_iters=5, tol=1e-300, lipschitz=float(d["L"]))
    est, _ = tf.solve_hierarchical(sino, tf.GridHierarchy(levels=(n,), iters_per_level=(5,)), prm,
                                   cfg)
    geom = tf.ScanGeometry(angles=d["angles"], detector_bins=d["g"].shape[2], image_side=n)
    p = tf.NufftPlan(n, tf.polar_sampling(geom), 1e-6)
    ctx = tf.fidelity_context(p, tf.build_psf(p.sampling, n), sino)
    rec, _ = tf.solve(ctx, prm, cfg, torch.zeros((d["g"].shape[0], n, n), device="cuda"))
    np.testing.assert_array_equal(est.data, rec.double().cpu().numpy())


@pytest.mark.parametrize("src,tgt", [((6, 40, 40), (12, 100)), ((3, 64, 64), (7, 128)),
                                     ((1, 25, 25), (1, 60)), ((5, 33, 33), (10, 300))])
def test_fused_upsample_matches_axis_passes(tf, rng, src, tgt):
    """K9f (all three axes in one pass) equals the per-axis K9 chain, for whole
    volumes and for slabs of the target read from a partial coarse source."""
    import torch

    from paper_2603_28756_b200.multires import (_resample_axis, _upsample3, slab_source_range,
                                                upsample_slab)

    x = torch.from_numpy(rng.standard_normal(src).astype(np.float32)).cuda()
    nz, side = tgt
    ref = _resample_axis(_resample_axis(_resample_axis(x, 0, nz), 1, side), 2, side)
    got = _upsample3(x, side, nz, 0, nz, src[0])
    assert got is not None
    assert float((got - ref).abs().max()) <= 1e-5 * float(ref.abs().max())
    for b, e in ((0, max(1, nz // 3)), (nz // 3, nz)):
        if b >= e:
            continue
        lo, hi = slab_source_range(src[0], nz, b, e)
        part = upsample_slab(x[lo:hi], side, nz, b, e, src_begin=lo, n_src=src[0])
        assert float((part - ref[b:e]).abs().max()) <= 1e-5 * float(ref.abs().max())
