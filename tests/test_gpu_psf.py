"""The PsfKernel / FidelityContext boundary against the reference's own kernel tests
(tests/test_toeplitz.py:63-94 of the reference, ported) and the NUFFT-of-ones
kernels stored in every tests/golden/toeplitz_*.npz (reference-generated)."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_28756_b200 as m

    return m


def _plan(tf, side, n_angles, bins=None, tol=1e-6):
    ang = np.linspace(0.0, np.pi, n_angles, endpoint=False)
    geom = tf.ScanGeometry(angles=ang, detector_bins=bins or side, image_side=side)
    samp = tf.polar_sampling(geom)
    return samp, tf.NufftPlan(side, samp, tol)


def _kernel(psf):
    return np.fft.fftshift(np.fft.ifft2(psf.spectrum)).real


def test_single_angle_matches_direct_summation(tf):
    """reference test_toeplitz.py:63-74."""
    from paper_2603_28756_b200.geometry import radial_frequencies

    geom = tf.ScanGeometry(angles=np.array([0.0]), detector_bins=4, image_side=4)
    samp = tf.polar_sampling(geom)
    psf = tf.compute_psf(tf.NufftPlan(7, samp, 1e-8), 4)
    assert psf.padded_side == 7 and psf.embed_offset == 1
    kernel = _kernel(psf)
    omega = radial_frequencies(4)
    lags = np.arange(7) - 3
    expected_x = np.array([np.sum(np.cos(omega * d)) for d in lags])
    np.testing.assert_allclose(kernel, expected_x[:, None] * np.ones((1, 7)),
                               atol=1e-6 * np.abs(expected_x).max())


def test_center_value_is_sample_count(tf):
    samp, _ = _plan(tf, 16, 9)
    psf = tf.build_psf(samp, 16)
    kernel = _kernel(psf)
    c = psf.padded_side // 2
    assert kernel[c, c] == pytest.approx(samp.count, rel=1e-6)


def test_centro_symmetry(tf):
    samp, _ = _plan(tf, 16, 9)
    kernel = _kernel(tf.build_psf(samp, 16))
    assert np.max(np.abs(kernel - kernel[::-1, ::-1])) <= 1e-6 * np.max(np.abs(kernel))


def test_spectrum_imaginary_part_small(tf):
    samp, _ = _plan(tf, 32, 11)
    psf = tf.build_psf(samp, 32)
    assert np.linalg.norm(psf.spectrum.imag) <= 1e-6 * np.linalg.norm(psf.spectrum)
    assert not psf.spectrum.flags.writeable


@pytest.mark.parametrize("path", sorted(glob.glob(str(GOLDEN / "toeplitz_*.npz"))),
                         ids=lambda p: os.path.basename(p))
def test_kernel_matches_reference_fixture(tf, path):
    """Closed-form fp64 kernel (K6 lags on the reference's odd grid) vs the reference's
    adjoint-NUFFT-of-ones kernel stored in the fixture (NUFFT tolerance 1e-6)."""
    d = dict(np.load(path))
    ang = d["angles"]
    nd = int(d["g"].shape[-1])
    side = int(d["f"].shape[-1])
    geom = tf.ScanGeometry(angles=ang, detector_bins=nd, image_side=side)
    psf = tf.build_psf(tf.polar_sampling(geom), side)
    assert psf.padded_side == int(d["padded_side"])
    assert psf.embed_offset == (int(d["padded_side"]) - side) // 2
    assert rel_l2(_kernel(psf), d["kernel"]) < 2e-6


def test_fidelity_context_reference_constructor(tf):
    """FidelityContext(psf, rstar_g=Volume|ImageGrid, g_norm_sq), as toeplitz.py:207 builds it."""
    d = golden("toeplitz_n64_p45_nd64_z2.npz")
    geom = tf.ScanGeometry(angles=d["angles"], detector_bins=64, image_side=64)
    psf = tf.build_psf(tf.polar_sampling(geom), 64)
    vol = tf.Volume(d["rstar"])
    ctx = tf.FidelityContext(psf=psf, rstar_g=vol, g_norm_sq=float(np.sum(d["g"] ** 2)))
    assert ctx.rstar_g is vol and ctx.slices == 2 and ctx.side == 64
    assert rel_l2(tf.fidelity_grad(ctx, d["f"]), d["grad"]) < 1e-4
    assert tf.fidelity_loss(ctx, d["f"]) == pytest.approx(float(d["loss"]), rel=1e-5)
    img = golden("toeplitz_n32_p45_nd32_z1.npz")
    geom = tf.ScanGeometry(angles=img["angles"], detector_bins=32, image_side=32)
    psf = tf.build_psf(tf.polar_sampling(geom), 32)
    ctx2 = tf.FidelityContext(psf, tf.ImageGrid(img["rstar"][0]), float(np.sum(img["g"] ** 2)))
    assert ctx2.slices == 1
    assert rel_l2(tf.fidelity_grad(ctx2, img["f"][0]), img["grad"][0]) < 1e-4
    with pytest.raises(AttributeError):
        ctx2.g_norm_sq = 0.0
    with pytest.raises(ValueError):
        tf.FidelityContext(psf, tf.ImageGrid(np.zeros((16, 16))), 0.0)
