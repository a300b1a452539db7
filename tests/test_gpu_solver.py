"""qGGMRF kernels and the GPU solver vs reference fixtures and the numpy oracle."""

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


def _ctx(tf, angles, g, n, f_rstar=None):
    """FidelityContext with R*g from the oracle (the NUFFT is tested separately)."""
    import torch

    import oracle as O

    nd = g.shape[-1]
    geom = tf.ScanGeometry(angles=angles, detector_bins=nd, image_side=n)
    psf = tf.build_psf(tf.polar_sampling(geom), n)
    rs = O.rstar(O.make_plan(n, angles, nd), g) if f_rstar is None else f_rstar
    return tf.FidelityContext(psf=psf, rstar=torch.from_numpy(rs.astype(np.float32)).cuda(),
                              g_norm_sq=float(np.sum(g ** 2)))


@pytest.mark.parametrize("name", ["qggmrf_s0.2_p2.0.npz", "qggmrf_s0.05_p1.8.npz"])
def test_prior_kernels_match_reference(tf, name):
    d = golden(name)
    sigma, lam, p, q, T = d["params"]
    prm = tf.QggmrfParams(sigma=sigma, lam=lam, p=p, q=q, T=T)
    s3, s2 = tf.stencil_3d(), tf.stencil_2d()
    assert rel_l2(tf.prior_grad(prm, s3, d["vol"]), d["grad"]) < 1e-5
    assert rel_l2(tf.prior_grad(prm, s3, d["vol"], halo_lo=d["lo"], halo_hi=d["hi"]),
                  d["grad_halo"]) < 1e-5
    assert tf.prior_energy(prm, s3, d["vol"]) == pytest.approx(float(d["energy"]), rel=1e-5)
    assert tf.prior_energy(prm, s3, d["vol"], halo_hi=d["hi"]) == pytest.approx(
        float(d["energy_halo"]), rel=1e-5)
    assert rel_l2(tf.prior_grad(prm, s2, d["img2"]), d["grad2"]) < 1e-5
    assert tf.prior_energy(prm, s2, d["img2"]) == pytest.approx(float(d["energy2"]), rel=1e-5)
    x = np.linspace(-3, 3, 61)
    np.testing.assert_allclose(tf.potential(prm, x), d["rho"], rtol=1e-12)
    np.testing.assert_allclose(tf.potential_deriv(prm, x), d["drho"], rtol=1e-12)


def test_constant_volume_zero_gradient(tf):
    prm = tf.QggmrfParams(sigma=0.3, lam=1.0)
    g = tf.prior_grad(prm, tf.stencil_3d(), np.full((4, 9, 9), 2.5))
    assert np.all(g == 0)


def test_split_with_halos_matches_unsplit(tf, rng):
    prm = tf.QggmrfParams(sigma=0.2, lam=1.0, p=2.0, q=1.1)
    vol = rng.standard_normal((6, 17, 19))
    s3 = tf.stencil_3d()
    full = tf.prior_grad(prm, s3, vol)
    top = tf.prior_grad(prm, s3, vol[:3], halo_hi=vol[3])
    bot = tf.prior_grad(prm, s3, vol[3:], halo_lo=vol[2])
    assert rel_l2(np.concatenate([top, bot]), full) < 1e-6
    e = tf.prior_energy(prm, s3, vol)
    e_split = tf.prior_energy(prm, s3, vol[:3], halo_hi=vol[3]) + tf.prior_energy(prm, s3, vol[3:])
    assert e_split == pytest.approx(e, rel=1e-6)


@pytest.mark.parametrize("name", ["solve_2d.npz", "solve_3d.npz"])
def test_solve_matches_reference(tf, name):
    d = golden(name)
    z, n = d["f0"].shape[0], d["f0"].shape[1]
    ctx = _ctx(tf, d["angles"], d["g"], n)
    prm = tf.QggmrfParams(sigma=float(d["sigma"]), lam=float(d["lam"]))
    cfg = tf.SolverConfig(max_iters=int(d["iters"]), tol=1e-300, lipschitz=float(d["L"]))
    f0 = d["f0"][0] if z == 1 else d["f0"]
    rec, recs = tf.solve(ctx, prm, cfg, f0)
    rec = np.asarray(rec).reshape(z, n, n)
    # reconstruction gate (BASELINE.json north star): relative L2 <= 1e-3
    assert rel_l2(rec, d["recon"]) < 1e-3
    assert [r.iter for r in recs] == list(range(int(d["iters"]) + 1))
    # objectives agree to fp32-gradient accuracy relative to the objective scale:
    # <f, Kf> carries ~1e-6 relative error (fp32 FFTs vs the reference's NUFFT kernel)
    obj = np.array([r.objective for r in recs])
    np.testing.assert_allclose(obj, d["objective"], rtol=1e-4, atol=1e-5 * abs(d["objective"][0]))
    assert rel_l2([r.grad_norm for r in recs], d["grad_norm"]) < 1e-4
    assert [r.restarted for r in recs] == list(d["restarted"])


def test_lipschitz_estimate(tf):
    d = golden("solve_2d.npz")
    ctx = _ctx(tf, d["angles"], d["g"], d["f0"].shape[1])
    prm = tf.QggmrfParams(sigma=float(d["sigma"]), lam=float(d["lam"]))
    assert tf.estimate_lipschitz(ctx.psf, prm) == pytest.approx(float(d["lipschitz_est"]), rel=1e-3)


def test_objective_and_first_step(tf):
    """One step from 0 with the prior off is exactly R*g / L (test_solver.py:111-121)."""
    d = golden("solve_2d.npz")
    n = d["f0"].shape[1]
    ctx = _ctx(tf, d["angles"], d["g"], n)
    prm = tf.QggmrfParams(sigma=1.0, lam=0.0)
    total, fid, prior = tf.objective(ctx, prm, np.zeros((n, n)))
    assert fid == pytest.approx(0.5 * float(np.sum(d["g"] ** 2)), rel=1e-12)
    assert prior == 0.0
    L = 1234.5
    rec, recs = tf.solve(ctx, prm, tf.SolverConfig(max_iters=1, lipschitz=L), np.zeros((n, n)))
    np.testing.assert_allclose(rec, ctx.rstar_array()[0] / L, rtol=1e-6, atol=1e-12)


def test_c1_reconstruction(tf):
    """C1 (256^2, 180 angles, Nd=512, FBP init, 100 iterations) vs the reference run."""
    d = golden("c1.npz")
    ctx = _ctx(tf, d["angles"], d["g"][None] if d["g"].ndim == 2 else d["g"], 256)
    prm = tf.QggmrfParams(sigma=float(d["sigma"]), lam=5e-4)
    cfg = tf.SolverConfig(max_iters=100, tol=1e-300, lipschitz=float(d["L"]))
    rec, recs = tf.solve(ctx, prm, cfg, d["f0"])
    assert rel_l2(rec, d["recon"]) < 1e-3
    # C1's objective is a ~1e-7 difference of ~1e7-sized terms (noisy data): fp32
    # K f carries ~1e-6 relative error, so records agree to ~1e-4 of obj_0
    np.testing.assert_allclose([r.objective for r in recs], d["objective"], rtol=1e-4,
                               atol=1e-4 * abs(d["objective"][0]))
    assert [r.restarted for r in recs] == list(d["restarted"])


def test_determinism_and_nonneg(tf):
    d = golden("solve_3d.npz")
    n = d["f0"].shape[1]
    ctx = _ctx(tf, d["angles"], d["g"], n)
    prm = tf.QggmrfParams(sigma=float(d["sigma"]), lam=float(d["lam"]))
    cfg = tf.SolverConfig(max_iters=6, tol=1e-300, lipschitz=float(d["L"]), nonneg=True)
    a, ra = tf.solve(ctx, prm, cfg, d["f0"])
    b, rb = tf.solve(ctx, prm, cfg, d["f0"])
    np.testing.assert_array_equal(a, b)
    assert [r.objective for r in ra] == [r.objective for r in rb]
    assert np.all(a >= 0)


def test_divergence_raises(tf):
    d = golden("solve_2d.npz")
    n = d["f0"].shape[1]
    ctx = _ctx(tf, d["angles"], d["g"], n)
    prm = tf.QggmrfParams(sigma=float(d["sigma"]), lam=float(d["lam"]))
    with pytest.raises(FloatingPointError):
        tf.solve(ctx, prm, tf.SolverConfig(max_iters=400, tol=1e-300, lipschitz=1e-6, restart=False),
                 d["f0"][0])


@pytest.mark.parametrize("shape", [(5, 72, 100), (3, 49, 161)])
def test_prior_kernels_interior_tiles(tf, rng, shape):
    """Slices larger than three K4/K5 tiles each way (interior + edge tiles, partial
    last tiles) against the oracle, for the gradient with both halos, the fused
    update and the energy / fidelity sums."""
    import torch

    import oracle as O

    prm = tf.QggmrfParams(sigma=0.3, lam=0.7, p=2.0, q=1.2, T=1.0)
    pr = O.Prior(sigma=0.3, lam=0.7)
    s3 = tf.stencil_3d()
    vol = rng.standard_normal(shape)
    lo, hi = rng.standard_normal(shape[1:]), rng.standard_normal(shape[1:])
    assert rel_l2(tf.prior_grad(prm, s3, vol, halo_lo=lo, halo_hi=hi),
                  O.prior_grad(pr, vol, halo_lo=lo, halo_hi=hi)) < 1e-5
    assert rel_l2(tf.prior_grad(prm, s3, vol), O.prior_grad(pr, vol)) < 1e-5
    assert tf.prior_energy(prm, s3, vol, halo_hi=hi) == pytest.approx(
        O.prior_energy(pr, vol, halo_hi=hi), rel=1e-5)
    # fused update: f_new = y - (K y - R*g + lam grad_prior(y)) / L, y = f + c (f - fp)
    from paper_2603_28756_b200.qggmrf import energy_fid, prior_update

    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()  # noqa: E731
    f, fp = vol, vol + 0.1 * rng.standard_normal(shape)
    kf, kfp, rs = (rng.standard_normal(shape) for _ in range(3))
    c, lam, inv_L = 0.4, 0.7, 0.05
    out = torch.empty(shape, dtype=torch.float32, device="cuda")
    gsq = prior_update(prm, s3, dev(f), dev(fp), out, kf=dev(kf), kfp=dev(kfp), rstar=dev(rs),
                       c=c, lam=lam, inv_L=inv_L)
    y = f + c * (f - fp)
    grad = kf + c * (kf - kfp) - rs + lam * O.prior_grad(O.Prior(sigma=0.3, lam=1.0), y)
    assert rel_l2(out.cpu().numpy(), y - inv_L * grad) < 1e-5
    assert float(gsq) == pytest.approx(float(np.sum(grad ** 2)), rel=1e-4)
    fn = out.cpu().numpy().astype(np.float64)
    kfn = rng.standard_normal(shape)
    e3 = energy_fid(prm, s3, dev(fn), f=dev(f), kfn=dev(kfn), kf=dev(kf), rstar=dev(rs)).cpu().numpy()
    assert e3[0] == pytest.approx(O.prior_energy(O.Prior(sigma=0.3), fn), rel=1e-5)
    assert e3[1] == pytest.approx(float(np.sum(fn * (0.5 * kfn - rs))), rel=1e-5, abs=1e-3)
    assert e3[2] == pytest.approx(float(np.sum((fn - f) * (0.5 * (kfn + kf) - rs))), rel=1e-5,
                                  abs=1e-3)


@pytest.mark.parametrize("shape", [(1, 5, 7), (2, 1, 33), (3, 40, 1), (2, 17, 2), (1, 33, 48)])
def test_prior_kernels_thin_slabs(tf, rng, shape):
    """Degenerate tiles (one-voxel-wide slices, single-slice slabs with both halos as in
    a distributed run with one slice per rank) against the oracle."""
    import oracle as O

    prm = tf.QggmrfParams(sigma=0.4, lam=1.0, p=1.8, q=1.1, T=1.3)
    pr = O.Prior(sigma=0.4, lam=1.0, p=1.8, q=1.1, T=1.3)
    s3 = tf.stencil_3d()
    vol = rng.standard_normal(shape)
    lo, hi = rng.standard_normal(shape[1:]), rng.standard_normal(shape[1:])
    got = tf.prior_grad(prm, s3, vol, halo_lo=lo, halo_hi=hi)
    assert rel_l2(got, O.prior_grad(pr, vol, halo_lo=lo, halo_hi=hi, three_d=True)) < 1e-5
    assert tf.prior_energy(prm, s3, vol, halo_hi=hi) == pytest.approx(
        O.prior_energy(pr, vol, halo_hi=hi, three_d=True), rel=1e-5)


def test_device_decision_matches_host_arithmetic(tf, rng):
    """tf_solver_decide reproduces the host loop's fp64 restart / momentum / stop
    arithmetic (solver.py:158-180) bit for bit, over restarts, convergence and
    non-finite objectives."""
    import math

    import torch

    from paper_2603_28756_b200.qggmrf import solver_decide

    lam, tol = 0.37, 1e-6
    state = torch.tensor([10.0, 9.0, 2.7, 1.0, 0.0], dtype=torch.float64, device="cuda")
    c_dev = torch.zeros(1, dtype=torch.float32, device="cuda")
    obj, fid, prior, t = 10.0, 9.0, 2.7, 1.0
    cases = [(rng.standard_normal(), abs(rng.standard_normal()), rng.standard_normal() * 1e-3)
             for _ in range(40)]
    # None: e_new = the CURRENT prior and dfid = 0, i.e. dobj = 0 -> converged; then inf
    cases += [None, (float("inf"), 1.0, -1.0)]
    n_conv = 0
    for restart in (True, False):
        for case in cases:
            e_new, gsq, dfid = (prior, 1.0, 0.0) if case is None else case
            vals = torch.tensor([e_new, gsq, dfid], dtype=torch.float64, device="cuda")
            rec = torch.empty(8, dtype=torch.float64, device="cuda")
            solver_decide(vals, state, c_dev, rec, lam=lam, with_prior=True, restart=restart,
                          tol=tol)
            r = rec.cpu().tolist()
            dobj = dfid + lam * (e_new - prior)
            obj_new = obj + dobj
            rst = restart and dobj > 0.0
            t_next = 1.0 if rst else (1.0 + math.sqrt(1.0 + 4.0 * t * t)) / 2.0
            c_next = 0.0 if rst else (t - 1.0) / t_next
            conv = (not rst) and abs(dobj) <= tol * abs(obj)
            fin = math.isfinite(obj_new)
            assert r[0] == obj_new or (not fin and not math.isfinite(r[0]))
            assert r[1] == fid + dfid and r[3] == gsq and r[7] == dobj or not fin
            assert bool(r[4]) == rst and bool(r[5]) == conv and bool(r[6]) == fin
            assert float(c_dev.item()) == float(np.float32(c_next)) or not fin
            n_conv += int(r[5])
            if case is None:
                assert r[7] == 0.0 and bool(r[5]), "zero increment must converge"
            if not fin:  # the solver raises here; restart the synthetic sequence
                state.copy_(torch.tensor([10.0, 9.0, 2.7, 1.0, 0.0], dtype=torch.float64))
                obj, fid, prior, t = 10.0, 9.0, 2.7, 1.0
                continue
            obj, fid, prior, t = obj_new, fid + dfid, e_new, t_next
    assert n_conv >= 2


def test_early_stop_records_and_snapshots(tf):
    """A realistic tolerance stops the solve early: the returned iterate, the records
    and the snapshots (k = 1 .. k_stop, no look-ahead iterate) agree with a fixed
    schedule of exactly k_stop iterations (solver.py:170-178)."""
    d = golden("solve_2d.npz")
    n = d["f0"].shape[1]
    ctx = _ctx(tf, d["angles"], d["g"], n)
    prm = tf.QggmrfParams(sigma=float(d["sigma"]), lam=float(d["lam"]))
    # a tolerance the fixed 30-iteration run crosses between iterations 5 and 20
    _, probe = tf.solve(ctx, prm, tf.SolverConfig(max_iters=30, tol=1e-300,
                                                  lipschitz=float(d["L"])), d["f0"][0])
    ratios = [abs(b.objective - a.objective) / abs(a.objective)
              for a, b in zip(probe, probe[1:]) if not b.restarted]
    tol = 1.5 * min(ratios[5:20])
    snaps = []
    cfg = tf.SolverConfig(max_iters=400, tol=tol, lipschitz=float(d["L"]))
    rec, recs = tf.solve(ctx, prm, cfg, d["f0"][0], snapshot_sink=lambda k, s: snaps.append((k, s)))
    k_stop = recs[-1].iter
    assert 1 < k_stop <= 21, "tolerance should stop the solve early"
    assert [r.iter for r in recs] == list(range(k_stop + 1))
    last = recs[-1]
    assert not last.restarted and abs(last.objective - recs[-2].objective) <= tol * abs(
        recs[-2].objective)
    assert [k for k, _ in snaps] == list(range(1, k_stop + 1))
    np.testing.assert_array_equal(snaps[-1][1].reshape(np.shape(rec)), rec)  # (1, n, n) as the reference
    fixed, frecs = tf.solve(ctx, prm, tf.SolverConfig(max_iters=k_stop, tol=1e-300,
                                                      lipschitz=float(d["L"])), d["f0"][0])
    np.testing.assert_array_equal(fixed, rec)
    assert [r.objective for r in frecs] == [r.objective for r in recs]


def test_divergence_sends_no_nonfinite_snapshot(tf):
    d = golden("solve_2d.npz")
    n = d["f0"].shape[1]
    ctx = _ctx(tf, d["angles"], d["g"], n)
    prm = tf.QggmrfParams(sigma=float(d["sigma"]), lam=float(d["lam"]))
    snaps = []
    with pytest.raises(FloatingPointError):
        tf.solve(ctx, prm, tf.SolverConfig(max_iters=400, tol=1e-300, lipschitz=1e-6,
                                           restart=False),
                 d["f0"][0], snapshot_sink=lambda k, s: snaps.append((k, s)))
    assert snaps and all(np.all(np.isfinite(s)) for _, s in snaps)
    assert [k for k, _ in snaps] == list(range(1, len(snaps) + 1))


def test_cuda_input_is_not_modified(tf):
    """solve copies a caller-owned CUDA f0 (solver.py:121); host inputs are converted
    into a buffer the loop owns."""
    import torch

    d = golden("solve_3d.npz")
    n = d["f0"].shape[1]
    ctx = _ctx(tf, d["angles"], d["g"], n)
    prm = tf.QggmrfParams(sigma=float(d["sigma"]), lam=float(d["lam"]))
    cfg = tf.SolverConfig(max_iters=5, tol=1e-300, lipschitz=float(d["L"]))
    f0 = torch.from_numpy(d["f0"].astype(np.float32)).cuda()
    keep = f0.clone()
    out, _ = tf.solve(ctx, prm, cfg, f0)
    assert torch.equal(f0, keep)
    host, _ = tf.solve(ctx, prm, cfg, d["f0"])
    np.testing.assert_array_equal(out.cpu().numpy().astype(np.float64), host)


@pytest.mark.parametrize("shape,halos", [((5, 72, 100), False), ((4, 49, 161), True),
                                         ((1, 33, 40), True)])
def test_fused_energy_update_matches_k5_k4(tf, rng, shape, halos):
    """K45 (tf_prior_energy_update) = K5's sums of f + K4's update at the no-restart
    momentum, bit for bit; the conditional re-run (tf_prior_update_if) is a no-op
    unless the restart flag is set, and then equals K4 at c = 0."""
    import math

    import torch

    from paper_2603_28756_b200.qggmrf import (energy_fid, prior_energy_update, prior_update,
                                              prior_update_if)

    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()  # noqa: E731
    prm = tf.QggmrfParams(sigma=0.3, lam=0.7, p=2.0, q=1.2, T=1.0)
    s3 = tf.stencil_3d()
    f, fp = dev(rng.standard_normal(shape)), dev(rng.standard_normal(shape))
    kf, kfp, rs = (dev(rng.standard_normal(shape)) for _ in range(3))
    pl = lambda: dev(rng.standard_normal(shape[1:])) if halos else None  # noqa: E731
    f_lo, f_hi, fp_lo, fp_hi = pl(), pl(), pl(), pl()
    if not halos:
        f_lo = f_hi = fp_lo = fp_hi = None
    t = 2.37
    state = torch.tensor([0.0, 0.0, 0.0, t, 0.0], dtype=torch.float64, device="cuda")
    t_next = (1.0 + math.sqrt(1.0 + 4.0 * t * t)) / 2.0
    c = float(np.float32((t - 1.0) / t_next))
    lam, inv_L = 0.7, 0.05
    ref_out = torch.empty_like(f)
    gsq_ref = prior_update(prm, s3, f, fp, ref_out, kf=kf, kfp=kfp, rstar=rs, c=c, lam=lam,
                           inv_L=inv_L, f_lo=f_lo, f_hi=f_hi, fp_lo=fp_lo, fp_hi=fp_hi)
    e3 = energy_fid(prm, s3, f, fn_hi=f_hi, f=fp, kfn=kf, kf=kfp, rstar=rs)
    out = kfp.clone()  # the solver writes over K f_prev
    kfp_in = kfp.clone()
    sums = torch.zeros(4, dtype=torch.float64, device="cuda")
    prior_energy_update(prm, s3, f, fp, out, kf=kf, kfp=out, rstar=rs, state=state, lam=lam,
                        inv_L=inv_L, f_lo=f_lo, f_hi=f_hi, fp_lo=fp_lo, fp_hi=fp_hi,
                        energy=sums[0], fid=sums[1], dfid=sums[2], gsq=sums[3])
    assert torch.equal(out, ref_out)
    got = sums.cpu().numpy()
    ref = e3.cpu().numpy()
    np.testing.assert_allclose(got[:3], ref, rtol=1e-12)
    assert got[3] == float(gsq_ref)
    assert torch.equal(kfp, kfp_in)
    # conditional re-run: flag 0 -> untouched; flag 1 -> K4 at y = f with c = *c_dev = 0
    flag = torch.zeros(1, dtype=torch.float64, device="cuda")
    c0 = torch.zeros(1, dtype=torch.float32, device="cuda")
    g2 = torch.full((1,), -1.0, dtype=torch.float64, device="cuda")
    prior_update_if(prm, s3, f, out, kf=kf, rstar=rs, c_dev=c0, only_if=flag[0], gsq_out=g2[0],
                    lam=lam, inv_L=inv_L, f_lo=f_lo, f_hi=f_hi)
    assert torch.equal(out, ref_out) and float(g2) == -1.0
    flag.fill_(1.0)
    prior_update_if(prm, s3, f, out, kf=kf, rstar=rs, c_dev=c0, only_if=flag[0], gsq_out=g2[0],
                    lam=lam, inv_L=inv_L, f_lo=f_lo, f_hi=f_hi)
    ref0 = torch.empty_like(f)
    gsq0 = prior_update(prm, s3, f, f, ref0, kf=kf, kfp=kf, rstar=rs, c=0.0, lam=lam,
                        inv_L=inv_L, f_lo=f_lo, f_hi=f_hi, fp_lo=f_lo, fp_hi=f_hi)
    assert torch.equal(out, ref0) and float(g2) == float(gsq0)
