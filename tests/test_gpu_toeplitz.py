"""CUDA Toeplitz path vs the reference (golden fixtures) and the numpy oracle."""

import glob
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, golden, rel_l2

pytestmark = pytest.mark.gpu

TOEPLITZ = sorted(Path(p).name for p in glob.glob(str(GOLDEN / "toeplitz_*.npz")))

# single gradient evaluation gate (BASELINE.json north star): relative L2 <= 1e-4
GRAD_TOL = 1e-4


@pytest.fixture(scope="module")
def tf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_28756_b200 as m

    return m


def _psf(tf, angles, nd, n):
    geom = tf.ScanGeometry(angles=angles, detector_bins=nd, image_side=n)
    return tf.build_psf(tf.polar_sampling(geom), n)


@pytest.mark.parametrize("name", TOEPLITZ)
def test_apply_matches_reference(tf, name):
    d = golden(name)
    n, nd = d["f"].shape[1], d["g"].shape[2]
    psf = _psf(tf, d["angles"], nd, n)
    out = tf.toeplitz_apply(psf, d["f"])
    assert out.dtype == np.float64 and out.shape == d["f"].shape
    assert rel_l2(out, d["kf"]) < 1e-5


@pytest.mark.parametrize("name", TOEPLITZ)
def test_grad_with_reference_rstar(tf, name):
    import torch

    d = golden(name)
    n, nd = d["f"].shape[1], d["g"].shape[2]
    psf = _psf(tf, d["angles"], nd, n)
    rs = torch.from_numpy(d["rstar"].astype(np.float32)).cuda()
    ctx = tf.FidelityContext(psf=psf, rstar=rs, g_norm_sq=float(np.sum(d["g"] ** 2)))
    grad = tf.fidelity_grad(ctx, d["f"])
    assert rel_l2(grad, d["grad"]) < GRAD_TOL
    assert tf.fidelity_loss(ctx, d["f"]) == pytest.approx(float(d["loss"]), rel=1e-5)


def test_zero_in_zero_out(tf):
    psf = _psf(tf, np.linspace(0, np.pi, 5, endpoint=False), 16, 16)
    out = tf.toeplitz_apply(psf, np.zeros((16, 16)))
    assert np.all(out == 0)


def test_self_adjoint_and_psd(tf, rng):
    psf = _psf(tf, np.linspace(0, np.pi, 9, endpoint=False), 24, 24)
    f, h = rng.standard_normal((2, 24, 24))
    lhs = np.sum(f * tf.toeplitz_apply(psf, h))
    rhs = np.sum(tf.toeplitz_apply(psf, f) * h)
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)
    for s in range(5):
        x = np.random.default_rng(s).standard_normal((24, 24))
        assert np.sum(x * tf.toeplitz_apply(psf, x)) >= -1e-6 * np.sum(x * x)


def test_batch_equals_slice_loop(tf, rng):
    psf = _psf(tf, np.linspace(0, np.pi, 5, endpoint=False), 16, 16)
    vol = rng.standard_normal((3, 16, 16))
    batch = tf.toeplitz_apply(psf, vol)
    for z in range(3):
        np.testing.assert_array_equal(batch[z], tf.toeplitz_apply(psf, vol[z]))


def test_size_mismatch(tf):
    psf = _psf(tf, np.linspace(0, np.pi, 5, endpoint=False), 16, 16)
    with pytest.raises(ValueError):
        tf.toeplitz_apply(psf, np.zeros((8, 8)))


@pytest.mark.parametrize("n,n_ang,nd", [(256, 90, 256), (512, 90, 1024), (200, 33, 201),
                                         (640, 60, 640), (600, 45, 601), (1280, 90, 1280)])
def test_apply_vs_oracle_midsize(tf, n, n_ang, nd):
    """Power-of-two sides and the 5 * 2^k sides of the radix-5 path (640, 600 -> 1280,
    1280 -> 2560)."""
    import oracle as O

    ang = np.linspace(0, np.pi, n_ang, endpoint=False)
    x = np.random.default_rng(n).standard_normal((2, n, n))
    ref = O.apply_batch(O.build_psf(ang, nd, n), x)
    psf = _psf(tf, ang, nd, n)
    assert psf.fft_side == _lib_side(n)
    out = tf.toeplitz_apply(psf, x)
    assert rel_l2(out, ref) < 1e-5


def _lib_side(n):
    m = 1
    while m < 2 * n - 1:
        m *= 2
    five = [5 * q for q in (256, 512, 1024) if 2 * n - 1 <= 5 * q < m]
    return five[0] if five else m


@pytest.mark.parametrize("nd", [2560, 2561])
def test_apply_2560_wedge_vs_oracle(tf, nd):
    """The C5 slice (configs[4]): one 2560^2 slice, 120 angles over a 120-degree wedge,
    on the radix-5 side M = 5120; Nd even (flip term) and odd."""
    import oracle as O

    n = 2560
    ang = np.linspace(0, 2 * np.pi / 3, 120, endpoint=False)
    x = np.random.default_rng(1).standard_normal((1, n, n))
    ref = O.apply_batch(O.build_psf(ang, nd, n), x)
    psf = _psf(tf, ang, nd, n)
    assert psf.fft_side == 5120
    out = tf.toeplitz_apply(psf, x)
    assert rel_l2(out, ref) < 1e-5


@pytest.mark.parametrize("nd", [2048, 2049])
def test_apply_2048_vs_oracle(tf, nd):
    """The bench size (C3/C4 slices): one 2048^2 slice, 128 angles, Nd = 2048 (even:
    flip term active) and 2049 (odd), SURVEY.md §8d."""
    import oracle as O

    n = 2048
    ang = np.linspace(0, np.pi, 128, endpoint=False)
    x = np.random.default_rng(0).standard_normal((1, n, n))
    ref = O.apply_batch(O.build_psf(ang, nd, n), x)
    out = tf.toeplitz_apply(_psf(tf, ang, nd, n), x)
    assert rel_l2(out, ref) < 1e-5


@pytest.mark.parametrize("nd", [2900])
def test_apply_8192_vs_oracle(tf, nd):
    """M = 8192 (2560 < N <= 4096): four-pass row transforms, so the mirror-pair
    last pass of K1 and first pass of K3 run after / before two exchanges."""
    import oracle as O

    n = 2900
    ang = np.linspace(0, np.pi, 16, endpoint=False)
    x = np.random.default_rng(3).standard_normal((1, n, n))
    ref = O.apply_batch(O.build_psf(ang, nd, n), x)
    psf = _psf(tf, ang, nd, n)
    assert psf.fft_side == 8192
    out = tf.toeplitz_apply(psf, x)
    assert rel_l2(out, ref) < 1e-5


def test_device_tensor_path(tf):
    import torch

    psf = _psf(tf, np.linspace(0, np.pi, 7, endpoint=False), 32, 32)
    x = torch.randn(4, 32, 32, device="cuda")
    y = tf.toeplitz_apply(psf, x)
    assert isinstance(y, torch.Tensor) and y.is_cuda and y.shape == x.shape
    ref = tf.toeplitz_apply(psf, x.double().cpu().numpy())
    assert rel_l2(y.double().cpu().numpy(), ref) < 1e-6


def test_repeated_apply_bitwise_stable(tf):
    """Async-race guard (TMA ring, bulk prefetch): 2048^2 applies repeated bit for bit."""
    import torch

    n = 2048
    psf = _psf(tf, np.linspace(0, np.pi, 16, endpoint=False), n, n)
    x = torch.randn((3, n, n), device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    ref = tf.toeplitz_apply(psf, x).clone()
    for _ in range(10):
        assert torch.equal(tf.toeplitz_apply(psf, x), ref)


@pytest.mark.parametrize("n,nd,z", [(700, 700, 1), (700, 701, 2), (1000, 1024, 5),
                                    (1400, 1400, 3), (1400, 1401, 6),
                                    # N % 4 != 0: partial last row block, per-thread
                                    # row stores instead of the bulk paths
                                    (1001, 1001, 2), (1022, 1024, 1)])
def test_apply_radix64_columns_vs_oracle(tf, n, nd, z):
    """The two-pass radix-64 column kernel (k_cols_conv64: M = 2048 for 640 < N <= 1024,
    M = 4096 for 1280 < N <= 2048): slice counts that leave some of its four
    per-CTA slice groups idle or unevenly loaded (z = 1, 2, 3, 5, 6), even and odd Nd."""
    import oracle as O

    ang = np.linspace(0, np.pi, 60, endpoint=False)
    x = np.random.default_rng(n + z).standard_normal((z, n, n))
    ref = O.apply_batch(O.build_psf(ang, nd, n), x)
    psf = _psf(tf, ang, nd, n)
    assert psf.fft_side == (2048 if n <= 1024 else 4096)
    out = tf.toeplitz_apply(psf, x)
    assert rel_l2(out, ref) < 1e-5
    for k in range(z):  # every slice, not just the stack as a whole
        assert rel_l2(out[k], ref[k]) < 1e-5
