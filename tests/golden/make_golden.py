"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports tomoforge from /root/reference/pkg/src (read-only, untouched) and
writes small ``.npz`` files next to this script.  The fixtures pin both the
numpy oracle (tests/test_oracle.py) and the CUDA path (tests/test_gpu_*.py,
which run on a GPU box where /root/reference does not exist).
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("TOMOFORGE_REF", "/root/reference/pkg/src"))
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    import tomoforge as tf
    from tomoforge import multires, qggmrf, runtime, solver, toeplitz

    def angles(n):
        return np.linspace(0.0, np.pi, n, endpoint=False)

    def setup(side, n_ang, bins, seed):
        geom = tf.ScanGeometry(angles=angles(n_ang), detector_bins=bins, image_side=side)
        samp = tf.polar_sampling(geom)
        plan = tf.NufftPlan(side, samp, 1e-6)
        psf = tf.build_psf(samp, side, 1e-6)
        rng = np.random.default_rng(seed)
        return geom, samp, plan, psf, rng

    # ---- Toeplitz apply / fidelity: (side, angles, bins, slices)
    for side, n_ang, bins, z in [(32, 45, 32, 1), (32, 45, 33, 1), (64, 45, 64, 2), (24, 9, 48, 3),
                                 (16, 6, 16, 1), (128, 60, 128, 1), (8, 6, 8, 1)]:
        geom, samp, plan, psf, rng = setup(side, n_ang, bins, seed=side + bins)
        f = rng.standard_normal((z, side, side))
        g = rng.standard_normal((z, n_ang, bins))
        sino = tf.Sinogram(angles=geom.angles, data=g)
        ctx = tf.fidelity_context(plan, psf, sino)
        np.savez_compressed(
            OUT / f"toeplitz_n{side}_p{n_ang}_nd{bins}_z{z}.npz",
            angles=geom.angles, f=f, g=g,
            kf=toeplitz._apply_batch(psf, f),
            rstar=ctx.rstar_array(),
            grad=np.asarray(tf.fidelity_grad(ctx, f)),
            loss=tf.fidelity_loss(ctx, f),
            fbp=np.asarray(tf.fbp(plan, sino).data),
            kernel=np.fft.fftshift(np.fft.ifft2(psf.spectrum)).real,
            padded_side=psf.padded_side,
        )

    # ---- forward projection (data synthesis) + type2/type1 pair
    geom, samp, plan, psf, rng = setup(32, 20, 40, seed=5)
    img = rng.standard_normal((32, 32))
    c = rng.standard_normal(samp.count) + 1j * rng.standard_normal(samp.count)
    np.savez_compressed(OUT / "nufft_n32_p20_nd40.npz", angles=geom.angles, img=img, c=c,
                        type2=tf.type2(plan, img), type1=tf.type1(plan, c),
                        proj=tf.forward_project(plan, img).data[0])

    # ---- qGGMRF prior
    rng = np.random.default_rng(11)
    vol = rng.standard_normal((5, 12, 14)) * 0.3
    lo, hi = rng.standard_normal((12, 14)), rng.standard_normal((12, 14))
    img2 = rng.standard_normal((1, 13, 13))
    for sigma, lam, p, q, T in [(0.2, 1e-2, 2.0, 1.2, 1.0), (0.05, 1.0, 1.8, 1.1, 0.7)]:
        prm = tf.QggmrfParams(sigma=sigma, lam=lam, p=p, q=q, T=T)
        s3, s2 = qggmrf.stencil_3d(), qggmrf.stencil_2d()
        np.savez_compressed(
            OUT / f"qggmrf_s{sigma}_p{p}.npz",
            params=np.array([sigma, lam, p, q, T]), vol=vol, lo=lo, hi=hi, img2=img2,
            grad=np.asarray(tf.prior_grad(prm, s3, vol)),
            grad_halo=np.asarray(tf.prior_grad(prm, s3, vol, halo_lo=lo, halo_hi=hi)),
            energy=tf.prior_energy(prm, s3, vol),
            energy_halo=tf.prior_energy(prm, s3, vol, halo_hi=hi),
            grad2=np.asarray(tf.prior_grad(prm, s2, img2)),
            energy2=tf.prior_energy(prm, s2, img2),
            rho=tf.potential(prm, np.linspace(-3, 3, 61)),
            drho=tf.potential_deriv(prm, np.linspace(-3, 3, 61)),
        )

    # ---- solver: 2D (FBP init, restart) and 3D with the prior
    for name, side, n_ang, bins, z, lam, iters in [("2d", 48, 30, 64, 1, 5e-3, 40),
                                                    ("3d", 24, 18, 32, 4, 2e-2, 25)]:
        geom, samp, plan, psf, rng = setup(side, n_ang, bins, seed=3)
        if z == 1:
            truth = tf.shepp_logan(side).data[None]
        else:
            truth = tf.shepp_logan(side, three_d=True, slices=z).data
        clean = np.stack([tf.forward_project(plan, s).data[0] for s in truth])
        g = clean + 0.05 * rng.standard_normal(clean.shape)
        sino = tf.Sinogram(angles=geom.angles, data=g)
        ctx = tf.fidelity_context(plan, psf, sino)
        f0 = tf.fbp(plan, sino)
        f0a = np.asarray(f0.data)
        sigma = 0.1 * float(f0a.max() - f0a.min())
        prm = tf.QggmrfParams(sigma=sigma, lam=lam)
        L = solver.estimate_lipschitz(psf, prm)
        cfg = tf.SolverConfig(max_iters=iters, tol=1e-300, lipschitz=L)
        rec, recs = tf.solve(ctx, prm, cfg, f0)
        np.savez_compressed(
            OUT / f"solve_{name}.npz", angles=geom.angles, g=g, f0=f0a.reshape(z, side, side),
            sigma=sigma, lam=lam, L=L, iters=iters,
            recon=np.asarray(rec.data).reshape(z, side, side),
            objective=np.array([r.objective for r in recs]),
            fidelity=np.array([r.fidelity for r in recs]),
            prior=np.array([r.prior for r in recs]),
            grad_norm=np.array([r.grad_norm for r in recs]),
            restarted=np.array([r.restarted for r in recs]),
            lipschitz_est=solver.estimate_lipschitz(psf, prm),
        )

    # ---- multires pieces
    rng = np.random.default_rng(21)
    v = rng.standard_normal((3, 10, 10))
    sino = tf.Sinogram(angles=angles(7), data=rng.standard_normal((6, 7, 37)))
    ds = multires.downsample_sinogram(sino, 4)
    np.savez_compressed(
        OUT / "multires.npz", v=v, up3=multires.upsample(v, 20, 6), up2=multires.upsample(v[0], 25),
        mat=multires._lanczos_matrix(10, 20, 3), mat_odd=multires._lanczos_matrix(7, 16, 3),
        sino=sino.data, ds_data=ds.data, ds_angles=ds.angles,
        ds_ang=multires.downsample_sinogram(sino, 2, downsample_angles=True).data,
        lanczos=multires.lanczos_kernel(np.linspace(-4, 4, 81)),
    )
    geom, samp, plan, psf, rng = setup(32, 16, 32, seed=8)
    truth = tf.shepp_logan(32, three_d=True, slices=4).data
    g = np.stack([tf.forward_project(plan, s).data[0] for s in truth])
    sino = tf.Sinogram(angles=geom.angles, data=g)
    prm = tf.QggmrfParams(sigma=0.1, lam=1e-2)
    hier = multires.GridHierarchy(levels=(16, 32), iters_per_level=(6, 4))
    est, lrecs = multires.solve_hierarchical(sino, hier, prm,
                                             tf.SolverConfig(max_iters=1, tol=1e-300),
                                             use_fbp_init=True)
    np.savez_compressed(OUT / "hier.npz", angles=geom.angles, g=g, recon=np.asarray(est.data),
                        obj0=np.array([r.objective for r in lrecs[0]]),
                        obj1=np.array([r.objective for r in lrecs[1]]))

    # ---- runtime: partition + distributed == single worker
    parts = {f"{n}_{w}": np.array([[p.begin, p.end] for p in runtime.partition(n, w)])
             for n, w in [(10, 3), (8, 4), (7, 7), (2048, 8), (13, 5)]}
    geom, samp, plan, psf, rng = setup(16, 10, 16, seed=9)
    g = rng.standard_normal((6, 10, 16))
    sino = tf.Sinogram(angles=geom.angles, data=g)
    prm = tf.QggmrfParams(sigma=0.3, lam=0.05)
    cfg = tf.SolverConfig(max_iters=8, tol=1e-300, lipschitz=None)
    vol2, recs2 = runtime.distributed_solve(sino, 16, prm, cfg, 2)
    vol1, recs1 = runtime.distributed_solve(sino, 16, prm, cfg, 1)
    np.savez_compressed(OUT / "runtime.npz", angles=geom.angles, g=g, recon_w2=vol2.data,
                        recon_w1=vol1.data, obj_w2=np.array([r.objective for r in recs2]),
                        obj_w1=np.array([r.objective for r in recs1]), **parts)

    # ---- C1 at reduced iteration count is too slow? no: 256^2, 180 angles, Nd=512
    if os.environ.get("GOLDEN_C1", "1") == "1":
        geom, samp, plan, psf, rng = setup(256, 180, 512, seed=7)
        truth = tf.shepp_logan(256).data
        clean = tf.forward_project(plan, truth).data
        g = clean + 0.5 * np.random.default_rng(7).standard_normal(clean.shape)
        sino = tf.Sinogram(angles=geom.angles, data=g)
        ctx = tf.fidelity_context(plan, psf, sino)
        f0 = tf.fbp(plan, sino)
        sigma = 0.1 * float(f0.data.max() - f0.data.min())
        prm = tf.QggmrfParams(sigma=sigma, lam=5e-4)
        L = solver.estimate_lipschitz(psf, prm)
        rec, recs = tf.solve(ctx, prm, tf.SolverConfig(max_iters=100, tol=1e-300, lipschitz=L), f0)
        np.savez_compressed(OUT / "c1.npz", angles=geom.angles, g=g.astype(np.float64),
                            f0=f0.data, sigma=sigma, L=L, recon=rec.data,
                            objective=np.array([r.objective for r in recs]),
                            restarted=np.array([r.restarted for r in recs]))
    print("golden fixtures written to", OUT)


def c2_reduced():
    """C2 (configs[1]) at reduced size: 4 x 128^2 Shepp-Logan, 90 sparse angles, Nd = 256,
    Poisson counts (harness-defined model: I0 = 1e4, mu = 2.5 / max(g),
    seed 0), qGGMRF lam = 5e-4, sigma = 0.1 range(FBP) ("auto"), 50 iterations, FBP init."""
    sys.path.insert(0, str(REF))
    import tomoforge as tf
    from tomoforge import solver

    side, n_ang, bins, z = 128, 90, 256, 4
    ang = np.linspace(0.0, np.pi, n_ang, endpoint=False)
    geom = tf.ScanGeometry(angles=ang, detector_bins=bins, image_side=side)
    samp = tf.polar_sampling(geom)
    plan = tf.NufftPlan(side, samp, 1e-6)
    psf = tf.build_psf(samp, side, 1e-6)
    truth = tf.shepp_logan(side, three_d=True, slices=z).data
    clean = np.stack([tf.forward_project(plan, s).data[0] for s in truth])
    i0, mu = 1e4, 2.5 / clean.max()
    counts = np.random.default_rng(0).poisson(i0 * np.exp(-mu * clean))
    g = -np.log(np.maximum(counts, 1) / i0) / mu
    sino = tf.Sinogram(angles=ang, data=g)
    ctx = tf.fidelity_context(plan, psf, sino)
    f0 = tf.fbp(plan, sino)
    sigma = 0.1 * float(f0.data.max() - f0.data.min())
    prm = tf.QggmrfParams(sigma=sigma, lam=5e-4)
    L = solver.estimate_lipschitz(psf, prm)
    rec, recs = tf.solve(ctx, prm, tf.SolverConfig(max_iters=50, tol=1e-300, lipschitz=L), f0)
    np.savez_compressed(OUT / "c2_reduced.npz", angles=ang, g=g, f0=f0.data, sigma=sigma, L=L,
                        recon=rec.data, objective=np.array([r.objective for r in recs]),
                        restarted=np.array([r.restarted for r in recs]))
    print("c2_reduced.npz written")


SUBSET = 1 << 18  # voxels kept of the large reconstructions (seeded uniform sample)


def _subset(vol: np.ndarray, seed: int) -> dict:
    """A fixed uniform sample of a large volume plus size-independent summaries:
    the relative L2 over 2^18 seeded voxels estimates the full-volume one."""
    flat = vol.reshape(-1)
    idx = np.sort(np.random.default_rng(seed).choice(flat.size, size=min(SUBSET, flat.size),
                                                     replace=False)).astype(np.int64)
    return {"idx": idx, "vals": flat[idx], "slice_norms": np.linalg.norm(vol, axis=(-2, -1)),
            "total_sum": float(vol.sum())}


def c2_full():
    """C2 (configs[1]) at its stated size: 16 x 512^2 3-D Shepp-Logan, 90 sparse angles,
    Nd = 1024, Poisson counts (I0 = 1e4, mu = 2.5 / max(g), seed 0),
    qGGMRF lam = 5e-4, sigma = 0.1 range(FBP) ("auto", cli.py:90-98), L by the
    reference's power iteration, 50 iterations, FBP init (solver.py:112-180).

    The sinogram is rounded to float32 BEFORE the reference runs, so the GPU test
    (which stores it as float32) sees bit-identical inputs."""
    sys.path.insert(0, str(REF))
    import tomoforge as tf
    from tomoforge import solver

    side, n_ang, bins, z = 512, 90, 1024, 16
    ang = np.linspace(0.0, np.pi, n_ang, endpoint=False)
    geom = tf.ScanGeometry(angles=ang, detector_bins=bins, image_side=side)
    samp = tf.polar_sampling(geom)
    plan = tf.NufftPlan(side, samp, 1e-6)
    psf = tf.build_psf(samp, side, 1e-6)
    truth = tf.shepp_logan(side, three_d=True, slices=z)
    clean = tf.project_volume(plan, truth).data
    i0, mu = 1e4, 2.5 / clean.max()
    counts = np.random.default_rng(0).poisson(i0 * np.exp(-mu * clean))
    g = (-np.log(np.maximum(counts, 1) / i0) / mu).astype(np.float32)
    sino = tf.Sinogram(angles=ang, data=g.astype(np.float64))
    ctx = tf.fidelity_context(plan, psf, sino)
    f0 = tf.fbp(plan, sino)
    sigma = 0.1 * float(f0.data.max() - f0.data.min())
    prm = tf.QggmrfParams(sigma=sigma, lam=5e-4)
    L = solver.estimate_lipschitz(psf, prm)
    rec, recs = tf.solve(ctx, prm, tf.SolverConfig(max_iters=50, tol=1e-300, lipschitz=L), f0)
    rs, fs = _subset(rec.data, 502), _subset(f0.data, 502)
    np.savez_compressed(OUT / "c2_full.npz", angles=ang, g=g, sigma=sigma, L=L,
                        recon_idx=rs["idx"], recon_vals=rs["vals"],
                        recon_slice_norms=rs["slice_norms"], recon_sum=rs["total_sum"],
                        f0_vals=fs["vals"], f0_slice_norms=fs["slice_norms"],
                        objective=np.array([r.objective for r in recs]),
                        restarted=np.array([r.restarted for r in recs]))
    print("c2_full.npz written")


def c3_chain():
    """C3 (configs[2]) geometry at its stated finest size: a slab of 8 of the 64 slices of
    the 2048^2 3-D Shepp-Logan (slices 28..35), 128 angles, Nd = 2048, the 3-level
    (512, 1024, 2048) Lanczos-3 schedule of multires.solve_hierarchical
    (multires.py:198-242) with FBP init and a reduced iteration budget (6, 3, 2).  The
    Lipschitz constant is left to the reference's per-level power iteration
    (cfg.lipschitz = None); the estimates are logged.  Slab z-downsampling gives
    2 -> 4 -> 8 slices over the levels (multires.py:123-124)."""
    sys.path.insert(0, str(REF))
    import time

    import tomoforge as tf
    from tomoforge import geometry, multires, solver

    side, n_ang, bins, z_total, z0, z = 2048, 128, 2048, 64, 28, 8
    ang = np.linspace(0.0, np.pi, n_ang, endpoint=False)
    geom = tf.ScanGeometry(angles=ang, detector_bins=bins, image_side=side)
    samp = tf.polar_sampling(geom)
    plan = tf.NufftPlan(side, samp, 1e-6)
    t0 = time.time()
    # the slab's slices of shepp_logan(2048, three_d=True, slices=64) (geometry.py:254-271)
    truth = np.zeros((z, side, side))
    for k in range(z):
        iz = z0 + k
        zc = (2.0 * iz - z_total + 1.0) / z_total
        scale = np.sqrt(max(0.0, 1.0 - (zc / geometry._Z_ENVELOPE) ** 2))
        truth[k] = geometry._rasterize_ellipses(side, axis_scale=scale)
    clean = tf.project_volume(plan, tf.Volume(truth)).data
    g = (clean + 0.5 * np.random.default_rng(33).standard_normal(clean.shape)).astype(np.float32)
    sino = tf.Sinogram(angles=ang, data=g.astype(np.float64))
    f_fbp = tf.fbp(plan, sino)
    sigma = 0.1 * float(f_fbp.data.max() - f_fbp.data.min())  # sigma "auto" (cli.py:90-98)
    print(f"c3: sinogram + fbp {time.time() - t0:.0f}s", flush=True)
    prm = tf.QggmrfParams(sigma=sigma, lam=5e-4)
    lips = []
    orig = solver.estimate_lipschitz

    def logged(psf, params):
        v = orig(psf, params)
        lips.append(v)
        return v

    solver.estimate_lipschitz = logged
    try:
        hier = multires.GridHierarchy(levels=(512, 1024, 2048), iters_per_level=(6, 3, 2))
        est, lrecs = multires.solve_hierarchical(sino, hier, prm,
                                                 tf.SolverConfig(max_iters=1, tol=1e-300),
                                                 use_fbp_init=True)
    finally:
        solver.estimate_lipschitz = orig
    print(f"c3: solve_hierarchical done {time.time() - t0:.0f}s", flush=True)
    rs = _subset(est.data, 503)
    np.savez_compressed(
        OUT / "c3_chain.npz", angles=ang, g=g, sigma=sigma, lipschitz=np.array(lips),
        iters=np.array(hier.iters_per_level), levels=np.array(hier.levels),
        recon_idx=rs["idx"], recon_vals=rs["vals"], recon_slice_norms=rs["slice_norms"],
        recon_sum=rs["total_sum"],
        **{f"objective{i}": np.array([r.objective for r in recs]) for i, recs in enumerate(lrecs)},
        **{f"restarted{i}": np.array([r.restarted for r in recs]) for i, recs in enumerate(lrecs)})
    print("c3_chain.npz written")


def c5_wedge():
    """C5 (configs[4]) geometry at reduced size: 4 x 320^2 3-D Shepp-Logan, 120 angles
    uniform in [0, 2 pi / 3) (limited-angle wedge), Nd = 320, Gaussian noise rms 0.5
    (seed 7), qGGMRF lam = 5e-4, sigma = 0.1 range(FBP), L by power iteration, 30
    iterations from FBP and from zero -- the reference's bench_init comparison
    (bench.py:108-131) on the wedge.  Float32-rounded sinogram, as c2_full."""
    sys.path.insert(0, str(REF))
    import tomoforge as tf
    from tomoforge import solver

    side, n_ang, bins, z = 320, 120, 320, 4
    ang = np.linspace(0.0, 2.0 * np.pi / 3.0, n_ang, endpoint=False)
    geom = tf.ScanGeometry(angles=ang, detector_bins=bins, image_side=side)
    samp = tf.polar_sampling(geom)
    plan = tf.NufftPlan(side, samp, 1e-6)
    psf = tf.build_psf(samp, side, 1e-6)
    truth = tf.shepp_logan(side, three_d=True, slices=z)
    clean = tf.project_volume(plan, truth).data
    g = (clean + 0.5 * np.random.default_rng(7).standard_normal(clean.shape)).astype(np.float32)
    sino = tf.Sinogram(angles=ang, data=g.astype(np.float64))
    ctx = tf.fidelity_context(plan, psf, sino)
    f_fbp = tf.fbp(plan, sino)
    sigma = 0.1 * float(f_fbp.data.max() - f_fbp.data.min())
    prm = tf.QggmrfParams(sigma=sigma, lam=5e-4)
    L = solver.estimate_lipschitz(psf, prm)
    cfg = tf.SolverConfig(max_iters=30, tol=1e-300, lipschitz=L)
    out = {"angles": ang, "g": g, "sigma": sigma, "L": L}
    for name, f0 in (("fbp", f_fbp), ("zero", tf.Volume(np.zeros((z, side, side))))):
        rec, recs = tf.solve(ctx, prm, cfg, f0)
        out[f"recon_{name}"] = rec.data.astype(np.float32)
        out[f"fidelity_{name}"] = np.array([r.fidelity for r in recs])
        out[f"objective_{name}"] = np.array([r.objective for r in recs])
        out[f"restarted_{name}"] = np.array([r.restarted for r in recs])
    np.savez_compressed(OUT / "c5_wedge.npz", **out)
    print("c5_wedge.npz written")


def fileio_fixtures():
    """Files written by the reference's fileio (tests/golden/fileio/): raw arrays with
    sidecars, a plan and its parse, a convergence CSV and a PGM preview."""
    sys.path.insert(0, str(REF))
    import dataclasses

    import tomoforge as tf
    from tomoforge import fileio
    from tomoforge.solver import IterationRecord

    out = OUT / "fileio"
    out.mkdir(exist_ok=True)
    rng = np.random.default_rng(31)
    fileio.save_array(out / "vol.raw", tf.Volume(rng.standard_normal((3, 5, 5)), pixel_size=0.5))
    fileio.save_array(out / "img.raw", tf.ImageGrid(rng.standard_normal((4, 4))))
    fileio.save_array(out / "sino.raw", tf.Sinogram(angles=np.linspace(0, np.pi, 6, endpoint=False),
                                                    data=rng.standard_normal((2, 6, 7))))
    (out / "plan.toml").write_text(
        "[geometry]\nimage_side = 64\n\n[qggmrf]\nsigma = \"auto\"\nlambda = 0.0005\np = 1.9\n\n"
        "[solver]\nmax_iters = 40\ntol = 1e-300\nlipschitz = 1234.5\nnonneg = true\n\n"
        "[hierarchy]\nlevels = 2\niters_per_level = [20, 10]\n\n[runtime]\nworkers = 2\nseed = 7\n\n"
        "[files]\ninit_volume = \"vol.raw\"\n")
    plan = fileio.load_plan(out / "plan.toml")
    fields = {k: (str(v) if isinstance(v, Path) else v) for k, v in dataclasses.asdict(plan).items()}
    fields["init_volume"] = Path(fields["init_volume"]).name
    (out / "plan_parsed.json").write_text(json.dumps(fields, indent=1, default=str))
    recs = [IterationRecord(i, 100.0 / (i + 1), 90.0 / (i + 1), 1.0 / 3, 0.5 ** i, 0.01 * i, i == 2)
            for i in range(4)]
    fileio.write_convergence_csv(out / "conv.csv", [(r, i % 2, 1) for i, r in enumerate(recs)],
                                 {"seed": 7, "image_side": 64, "init": "fbp"})
    img = tf.ImageGrid(np.outer(np.arange(6.0), np.ones(6)))
    fileio.export_slice(out / "prev.pgm", img)
    print("fileio fixtures written")


def bench_csvs():
    """The reference's bench categories at small sizes (CSV files as the reference
    writes them): toeplitz (direct vs Toeplitz) and init (FBP vs zero)."""
    sys.path.insert(0, str(REF))
    from tomoforge import bench as rb

    out = OUT / "bench"
    out.mkdir(exist_ok=True)
    rb.bench_toeplitz(out / "toeplitz.csv", sizes=(32, 48), n_angles=20, seed=0, repeats=1)
    rb.bench_init(out / "init.csv", side=64, n_angles=30, max_iters=20, seed=7)
    rb.bench_multires(out / "multires.csv", side=64, n_angles=30, single_iters=40,
                      fine_iters=8, seed=7)
    print("bench csv fixtures written")


if __name__ == "__main__":
    if "--only-bench" in sys.argv:
        bench_csvs()
    elif "--only-c2" in sys.argv:
        c2_reduced()
    elif "--only-fileio" in sys.argv:
        fileio_fixtures()
    elif "--only-c2-full" in sys.argv:
        c2_full()
    elif "--only-c3" in sys.argv:
        c3_chain()
    elif "--only-c5" in sys.argv:
        c5_wedge()
    else:
        main()
        c2_reduced()
        fileio_fixtures()
