"""CUDA NUFFT back-projection / ramp filter / FBP vs reference fixtures and the oracle."""

import glob
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, golden, rel_l2

pytestmark = pytest.mark.gpu

TOEPLITZ = sorted(Path(p).name for p in glob.glob(str(GOLDEN / "toeplitz_*.npz")))


@pytest.fixture(scope="module")
def tf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_28756_b200 as m

    return m


def _plan(tf, angles, nd, n):
    geom = tf.ScanGeometry(angles=angles, detector_bins=nd, image_side=n)
    return tf.NufftPlan(n, tf.polar_sampling(geom), 1e-6)


@pytest.mark.parametrize("name", TOEPLITZ)
def test_rstar_and_fbp_match_reference(tf, name):
    d = golden(name)
    n, nd = d["f"].shape[1], d["g"].shape[2]
    p = _plan(tf, d["angles"], nd, n)
    sino = tf.Sinogram(angles=d["angles"], data=d["g"])
    psf = tf.build_psf(p.sampling, n)
    ctx = tf.fidelity_context(p, psf, sino)
    assert rel_l2(ctx.rstar_array(), d["rstar"]) < 1e-5
    assert ctx.g_norm_sq == pytest.approx(float(np.sum(d["g"] ** 2)), rel=1e-12)
    rec = tf.fbp(p, sino)
    assert rel_l2(np.asarray(rec.data).reshape(d["fbp"].shape), d["fbp"]) < 1e-5
    # the full fidelity gradient now runs on the GPU end to end
    assert rel_l2(tf.fidelity_grad(ctx, d["f"]), d["grad"]) < 1e-4


def test_type1_matches_reference(tf):
    d = golden("nufft_n32_p20_nd40.npz")
    p = _plan(tf, d["angles"], 40, 32)
    out = tf.type1(p, d["c"])
    assert out.dtype == np.complex128 and out.shape == (32, 32)
    assert rel_l2(out, d["type1"]) < 1e-5


@pytest.mark.parametrize("nd", [32, 33, 40, 256, 2560])
def test_ramp_filter_apply(tf, nd):
    import oracle as O

    ang = np.linspace(0, np.pi, 7, endpoint=False)
    data = np.random.default_rng(nd).standard_normal((2, 7, nd))
    out = tf.ramp_filter_apply(tf.Sinogram(angles=ang, data=data))
    assert rel_l2(out.data, O.ramp_filter_apply(data)) < 1e-5


def test_zero_sinogram(tf):
    ang = np.linspace(0, np.pi, 12, endpoint=False)
    p = _plan(tf, ang, 32, 32)
    assert np.all(tf.fbp(p, tf.Sinogram(angles=ang, data=np.zeros((12, 32)))).data == 0)


def test_fbp_shepp_logan_correlation(tf):
    """Frozen NCC of the reference (test_radon.py:185-193)."""
    import oracle as O

    n, n_ang, nd = 128, 60, 256
    ang = np.linspace(0, np.pi, n_ang, endpoint=False)
    phantom = tf.shepp_logan(n).data
    sino = O.forward_project(O.make_plan(n, ang, nd), phantom)
    rec = tf.fbp(_plan(tf, ang, nd, n), tf.Sinogram(angles=ang, data=sino)).data
    a, b = rec - rec.mean(), phantom - phantom.mean()
    ncc = np.sum(a * b) / np.sqrt(np.sum(a * a) * np.sum(b * b))
    assert ncc == pytest.approx(0.9299, abs=0.02)


def test_fbp_disk_interior(tf):
    """test_radon.py:171-183"""
    import oracle as O

    n, n_ang, nd = 128, 180, 256
    ang = np.linspace(0, np.pi, n_ang, endpoint=False)
    disk = tf.disk_phantom(n, 32.0).data
    sino = O.forward_project(O.make_plan(n, ang, nd), disk)
    rec = tf.fbp(_plan(tf, ang, nd, n), tf.Sinogram(angles=ang, data=sino)).data
    x = np.arange(n) - (n - 1) / 2.0
    interior = x[:, None] ** 2 + x[None, :] ** 2 < 30.0 ** 2
    assert np.sqrt(np.mean((rec[interior] - 1.0) ** 2)) <= 0.05


@pytest.mark.parametrize("n,n_ang,nd", [(200, 33, 201), (256, 90, 512), (2048, 128, 2048)])
def test_back_project_vs_oracle(tf, n, n_ang, nd):
    import oracle as O

    ang = np.linspace(0, np.pi, n_ang, endpoint=False)
    g = np.random.default_rng(n).standard_normal((1, n_ang, nd))
    ref = O.rstar(O.make_plan(n, ang, nd), g)
    p = _plan(tf, ang, nd, n)
    got = tf.back_project(p, tf.Sinogram(angles=ang, data=g)).data
    assert rel_l2(got, ref[0]) < 1e-5


def test_back_project_deterministic_and_batched(tf):
    from paper_2603_28756_b200.radon import back_project_stack

    ang = np.linspace(0, np.pi, 30, endpoint=False)
    g = np.random.default_rng(3).standard_normal((5, 30, 64))
    p = _plan(tf, ang, 64, 64)
    a = back_project_stack(p, g).cpu().numpy()
    b = back_project_stack(p, g).cpu().numpy()
    np.testing.assert_array_equal(a, b)
    for z in range(5):
        np.testing.assert_array_equal(a[z], back_project_stack(p, g[z:z + 1]).cpu().numpy()[0])


def test_sampling_mismatch_raises(tf):
    ang = np.linspace(0, np.pi, 12, endpoint=False)
    p = _plan(tf, ang, 32, 32)
    with pytest.raises(ValueError):
        tf.fbp(p, tf.Sinogram(angles=ang, data=np.zeros((12, 33))))


def test_device_plan_weights_match_host(tf):
    ang = np.linspace(0, np.pi, 40, endpoint=False)
    p = _plan(tf, ang, 200, 100)
    host = p.tables
    dev = p.device_tables()
    np.testing.assert_array_equal(dev["ab"].cpu().numpy(), host.ab)
    np.testing.assert_allclose(dev["wts"].cpu().numpy(), host.wts, rtol=2e-6, atol=1e-6)


def test_type2_and_forward_project_match_reference(tf):
    d = golden("nufft_n32_p20_nd40.npz")
    p = _plan(tf, d["angles"], 40, 32)
    assert rel_l2(tf.type2(p, d["img"]), d["type2"]) < 1e-5
    proj = tf.forward_project(p, d["img"])
    assert rel_l2(proj.data[0], d["proj"]) < 1e-5


@pytest.mark.parametrize("n,n_ang,nd", [(33, 10, 33), (128, 60, 256), (2048, 128, 2048)])
def test_forward_project_vs_oracle(tf, n, n_ang, nd):
    import oracle as O

    ang = np.linspace(0, np.pi, n_ang, endpoint=False)
    img = np.random.default_rng(n).standard_normal((n, n))
    ref = O.forward_project(O.make_plan(n, ang, nd), img)
    got = tf.forward_project(_plan(tf, ang, nd, n), img).data[0]
    assert rel_l2(got, ref) < 1e-5


def test_projector_adjointness(tf):
    """<R f, g> = <f, R* g> on the GPU pair (test_radon.py:113-120)."""
    from paper_2603_28756_b200.radon import back_project_stack, forward_project_stack

    ang = np.linspace(0, np.pi, 45, endpoint=False)
    p = _plan(tf, ang, 96, 64)
    rng = np.random.default_rng(9)
    f, g = rng.standard_normal((3, 64, 64)), rng.standard_normal((3, 45, 96))
    rf = forward_project_stack(p, f).double().cpu().numpy()
    rtg = back_project_stack(p, g).double().cpu().numpy()
    lhs, rhs = np.sum(rf * g), np.sum(f * rtg)
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


def test_direct_dft_matches_reference_type2(tf):
    """The fp64 brute-force sum agrees with the reference's type2 to its tolerance
    (test_nufft.py:70-85) and with our type2."""
    d = golden("nufft_n32_p20_nd40.npz")
    p = _plan(tf, d["angles"], 40, 32)
    direct = tf.direct_dft(p.sampling, d["img"])
    assert rel_l2(d["type2"], direct) < 1e-6
    assert rel_l2(tf.type2(p, d["img"]), direct) < 1e-5
    with pytest.raises(ValueError):
        tf.direct_dft(p.sampling, np.zeros((130, 130)))
