"""The numpy oracle against fixtures produced by the reference itself (CPU only)."""

import glob
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, golden, rel_l2

TOEPLITZ = sorted(Path(p).name for p in glob.glob(str(GOLDEN / "toeplitz_*.npz")))


@pytest.mark.parametrize("name", TOEPLITZ)
def test_toeplitz_fixture(name):
    d = golden(name)
    z, n = d["f"].shape[0], d["f"].shape[1]
    nd = d["g"].shape[2]
    psf = O.build_psf(d["angles"], nd, n)
    assert psf.m == int(d["padded_side"])
    np.testing.assert_allclose(O.apply_batch(psf, d["f"]), d["kf"], rtol=0, atol=1e-10 * np.abs(d["kf"]).max())
    plan = O.make_plan(n, d["angles"], nd)
    rs = O.rstar(plan, d["g"])
    assert rel_l2(rs, d["rstar"]) < 1e-12
    assert rel_l2(O.fidelity_grad(psf, rs, d["f"]), d["grad"]) < 1e-12
    assert O.fidelity_loss(psf, rs, float(np.sum(d["g"] ** 2)), d["f"]) == pytest.approx(float(d["loss"]), rel=1e-12)
    assert rel_l2(O.fbp(plan, d["g"]), d["fbp"]) < 1e-12


def test_nufft_fixture():
    d = golden("nufft_n32_p20_nd40.npz")
    p = O.make_plan(32, d["angles"], 40)
    assert rel_l2(O.type2(p, d["img"]), d["type2"]) < 1e-13
    assert rel_l2(O.type1(p, d["c"]), d["type1"]) < 1e-13
    assert rel_l2(O.forward_project(p, d["img"]), d["proj"]) < 1e-13


@pytest.mark.parametrize("name", ["qggmrf_s0.2_p2.0.npz", "qggmrf_s0.05_p1.8.npz"])
def test_qggmrf_fixture(name):
    d = golden(name)
    sigma, lam, p, q, T = d["params"]
    pr = O.Prior(sigma=sigma, lam=lam, p=p, q=q, T=T)
    assert rel_l2(O.prior_grad(pr, d["vol"]), d["grad"]) < 1e-13
    assert rel_l2(O.prior_grad(pr, d["vol"], d["lo"], d["hi"]), d["grad_halo"]) < 1e-13
    assert O.prior_energy(pr, d["vol"]) == pytest.approx(float(d["energy"]), rel=1e-13)
    assert O.prior_energy(pr, d["vol"], d["hi"]) == pytest.approx(float(d["energy_halo"]), rel=1e-13)
    assert rel_l2(O.prior_grad(pr, d["img2"]), d["grad2"]) < 1e-13
    assert O.prior_energy(pr, d["img2"]) == pytest.approx(float(d["energy2"]), rel=1e-13)
    x = np.linspace(-3, 3, 61)
    np.testing.assert_allclose(O.rho(pr, x), d["rho"], rtol=1e-14)
    np.testing.assert_allclose(O.rho_prime(pr, x), d["drho"], rtol=1e-14)


@pytest.mark.parametrize("name", ["solve_2d.npz", "solve_3d.npz"])
def test_solver_fixture(name):
    d = golden(name)
    z, n = d["f0"].shape[0], d["f0"].shape[1]
    nd = d["g"].shape[2]
    psf = O.build_psf(d["angles"], nd, n)
    plan = O.make_plan(n, d["angles"], nd)
    rs = O.rstar(plan, d["g"])
    pr = O.Prior(sigma=float(d["sigma"]), lam=float(d["lam"]))
    assert O.estimate_lipschitz(psf, pr) == pytest.approx(float(d["lipschitz_est"]), rel=1e-12)
    f0 = O.fbp(plan, d["g"])
    assert rel_l2(f0, d["f0"]) < 1e-12
    rec, recs = O.solve(psf, rs, float(np.sum(d["g"] ** 2)), pr, f0, int(d["iters"]), float(d["L"]), tol=1e-300)
    assert rel_l2(rec, d["recon"]) < 1e-10
    np.testing.assert_allclose([r.objective for r in recs], d["objective"], rtol=1e-10)
    assert [r.restarted for r in recs] == list(d["restarted"])


def test_multires_fixture():
    d = golden("multires.npz")
    assert rel_l2(O.upsample(d["v"], 20, 6), d["up3"]) < 1e-13
    assert rel_l2(O.upsample(d["v"][0], 25), d["up2"]) < 1e-13
    np.testing.assert_allclose(O.lanczos_matrix(10, 20), d["mat"], atol=1e-15)
    np.testing.assert_allclose(O.lanczos_matrix(7, 16), d["mat_odd"], atol=1e-15)
    ang = np.linspace(0, np.pi, 7, endpoint=False)
    a, ds = O.downsample_sinogram(ang, d["sino"], 4)
    np.testing.assert_array_equal(ds, d["ds_data"])
    _, dsa = O.downsample_sinogram(ang, d["sino"], 2, downsample_angles=True)
    np.testing.assert_array_equal(dsa, d["ds_ang"])
    np.testing.assert_allclose(O.lanczos(np.linspace(-4, 4, 81)), d["lanczos"], atol=1e-15)


def test_hierarchical_fixture():
    d = golden("hier.npz")
    pr = O.Prior(sigma=0.1, lam=1e-2)
    est, recs = O.solve_hierarchical(d["angles"], d["g"], (16, 32), (6, 4), pr, use_fbp_init=True)
    assert rel_l2(est, d["recon"]) < 1e-10
    np.testing.assert_allclose([r.objective for r in recs[1]], d["obj1"], rtol=1e-10)


def test_partition_fixture():
    d = golden("runtime.npz")
    for key in ("10_3", "8_4", "7_7", "2048_8", "13_5"):
        n, w = map(int, key.split("_"))
        assert np.array_equal(np.array(O.partition(n, w)), d[key])
    np.testing.assert_allclose(d["recon_w2"], d["recon_w1"], atol=1e-10)


def test_c2_reduced_fixture():
    """The oracle reproduces the reference's C2 (reduced, Poisson) run."""
    d = golden("c2_reduced.npz")
    n = d["f0"].shape[-1]
    nd = d["g"].shape[2]
    psf = O.build_psf(d["angles"], nd, n)
    plan = O.make_plan(n, d["angles"], nd)
    assert rel_l2(O.fbp(plan, d["g"]), d["f0"]) < 1e-12
    rs = O.rstar(plan, d["g"])
    pr = O.Prior(sigma=float(d["sigma"]), lam=5e-4)
    rec, recs = O.solve(psf, rs, float(np.sum(d["g"] ** 2)), pr, d["f0"], 50, float(d["L"]),
                        tol=1e-300)
    assert rel_l2(rec, d["recon"]) < 1e-10
    assert [r.restarted for r in recs] == list(d["restarted"])
