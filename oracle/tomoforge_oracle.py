"""float64 numpy restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Each function names the reference lines (pkg/src/tomoforge/<file>:<lines>) it
restates.  Written for clarity, not speed, except ``apply_batch`` which keeps
the reference's own FFT algorithm (complex fft2 on the odd 7-smooth padded
grid) because it doubles as the timed CPU baseline in bench.py.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, replace

import numpy as np

# ----------------------------------------------------------------- geometry
# geometry.py:196-213


def signed_bins(nd: int) -> np.ndarray:
    return np.arange(-(nd // 2), (nd + 1) // 2)


def radial_frequencies(nd: int) -> np.ndarray:
    return 2.0 * np.pi * signed_bins(nd) / nd


def polar_samples(angles: np.ndarray, nd: int) -> np.ndarray:
    """(P*Nd, 2) samples (w cos t, w sin t), angle-major (geometry.py:204-213)."""
    w = radial_frequencies(nd)
    return np.stack([np.outer(np.cos(angles), w).ravel(), np.outer(np.sin(angles), w).ravel()], 1)


def nyquist_mask(n_angles: int, nd: int) -> np.ndarray:
    """geometry.py:186-193"""
    if nd % 2:
        return np.zeros(n_angles * nd, dtype=bool)
    return np.tile(signed_bins(nd) == -(nd // 2), n_angles)


def uniform_angles(count: int) -> np.ndarray:
    return np.linspace(0.0, np.pi, count, endpoint=False)


# ------------------------------------------------------------------- NUFFT
# nufft.py:38-223

TABLE_PER_UNIT = 16384
_GAMMA = {3: 0.94, 4: 0.96, 5: 0.97, 6: 0.98, 7: 0.985}


def kernel_width(tol: float) -> int:
    """nufft.py:54-57"""
    return max(2, int(math.ceil(-math.log10(tol) - 1e-9)) + 1)


def kb_beta(width: int, sigma: float) -> float:
    """nufft.py:128-129"""
    return _GAMMA.get(width, 0.99) * math.pi * width * (1.0 - 1.0 / (2.0 * sigma))


def kb_table(width: int, beta: float):
    """Lookup table of I0(beta sqrt(1-(2x/w)^2)) on [0, w/2] (nufft.py:80-87)."""
    n_tab = int(width / 2 * TABLE_PER_UNIT) + 2
    step = (width / 2) / (n_tab - 2)
    x = np.arange(n_tab) * step
    arg = 1.0 - (2.0 * x / width) ** 2
    tab = np.where(arg > 0, np.i0(beta * np.sqrt(np.clip(arg, 0, None))), 0.0)
    return tab, step


def kb_eval(tab: np.ndarray, step: float, x: np.ndarray) -> np.ndarray:
    """Linear interpolation in the table, zero off support (nufft.py:69-77)."""
    t = np.abs(x) / step
    i = t.astype(np.int64)
    ok = i < tab.size - 1
    i = np.where(ok, i, 0)
    fr = t - i
    return np.where(ok, tab[i] * (1.0 - fr) + tab[i + 1] * fr, 0.0)


def kb_fourier(xi, width: int, beta: float) -> np.ndarray:
    """Closed-form KB transform (nufft.py:90-101)."""
    z = beta * beta - (np.pi * width * np.asarray(xi, dtype=np.float64)) ** 2
    r = np.sqrt(np.abs(z))
    safe = np.where(r == 0, 1.0, r)
    val = np.where(z > 0, np.sinh(r) / safe, np.sin(r) / safe)
    return width * np.where(r == 0, 1.0, val)


@dataclass
class Plan:
    """NUFFT plan (nufft.py:104-168)."""

    n: int
    os: int
    width: int
    beta: float
    deapod: np.ndarray
    phase: np.ndarray
    ix: np.ndarray
    wx: np.ndarray
    iy: np.ndarray
    wy: np.ndarray
    embed: int
    samples: np.ndarray
    angles: np.ndarray
    nd: int


def make_plan(n: int, angles: np.ndarray, nd: int, tol: float = 1e-6, sigma: float = 2.0) -> Plan:
    angles = np.asarray(angles, dtype=np.float64)
    samples = polar_samples(angles, nd)
    w = kernel_width(tol)
    beta = kb_beta(w, sigma)
    tab, step = kb_table(w, beta)
    os_ = int(math.ceil(sigma * n))
    os_ += os_ % 2
    xp = np.arange(n) - n // 2
    dk = kb_fourier(xp / os_, w, beta)
    lo = 1e-12 * np.abs(dk).max()
    dk = np.where(np.abs(dk) < lo, lo, dk)
    shift = n // 2 - (n - 1) / 2.0
    kx, ky = samples[:, 0], samples[:, 1]
    phase = np.exp(-1j * (kx + ky) * shift)

    def windows(k):
        eta = k * os_ / (2.0 * np.pi)
        first = np.ceil(eta - w / 2.0).astype(np.int64)
        idx = first[:, None] + np.arange(w)[None, :]
        return idx % os_, kb_eval(tab, step, idx - eta[:, None])

    ix, wx = windows(kx)
    iy, wy = windows(ky)
    return Plan(n, os_, w, beta, 1.0 / dk, phase, ix, wx, iy, wy, os_ // 2 - n // 2, samples,
                angles, nd)


def type1(p: Plan, c: np.ndarray) -> np.ndarray:
    """samples -> (n, n) complex grid (nufft.py:203-223)."""
    c = np.asarray(c, dtype=np.complex128) * np.conj(p.phase)
    vals = (p.wx[:, :, None] * p.wy[:, None, :]) * c[:, None, None]
    flat = (p.ix[:, :, None] * p.os + p.iy[:, None, :]).ravel()
    size = p.os * p.os
    grid = (np.bincount(flat, vals.real.ravel(), size)
            + 1j * np.bincount(flat, vals.imag.ravel(), size)).reshape(p.os, p.os)
    g = np.fft.fftshift(np.fft.ifft2(grid)) * size
    e = p.embed
    return g[e:e + p.n, e:e + p.n] * np.outer(p.deapod, p.deapod)


def type2(p: Plan, img: np.ndarray) -> np.ndarray:
    """(n, n) grid -> samples (nufft.py:184-200)."""
    pad = np.zeros((p.os, p.os), dtype=np.complex128)
    e = p.embed
    pad[e:e + p.n, e:e + p.n] = img * np.outer(p.deapod, p.deapod)
    G = np.fft.fft2(np.fft.ifftshift(pad))
    vals = G[p.ix[:, :, None], p.iy[:, None, :]]
    return np.einsum("mi,mj,mij->m", p.wx, p.wy, vals) * p.phase


# ------------------------------------------------------------------- radon
# radon.py:50-160


def detector_phase(nd: int) -> np.ndarray:
    return np.exp(-1j * radial_frequencies(nd) * (nd - 1) / 2.0)


def forward_project(p: Plan, img: np.ndarray) -> np.ndarray:
    """(n, n) -> (P, Nd) rows (radon.py:85-96)."""
    spec = type2(p, img).reshape(p.angles.size, p.nd) * detector_phase(p.nd)[None]
    return np.fft.ifft(np.fft.ifftshift(spec, axes=1), axis=1).real


def back_project_rows(p: Plan, rows: np.ndarray) -> np.ndarray:
    """(P, Nd) -> (n, n) adjoint (radon.py:124-128)."""
    nd = rows.shape[-1]
    spec = np.fft.fftshift(np.fft.fft(rows, axis=1), axes=1)
    return type1(p, (spec * np.conj(detector_phase(nd))[None] / nd).ravel()).real


def ramp_filter_apply(data: np.ndarray) -> np.ndarray:
    """(..., Nd) circular |w| filter (radon.py:137-142)."""
    nd = data.shape[-1]
    h = np.fft.ifftshift(np.abs(radial_frequencies(nd)))
    return np.fft.ifft(np.fft.fft(data, axis=-1) * h, axis=-1).real


def fbp(p: Plan, sino: np.ndarray) -> np.ndarray:
    """(Z, P, Nd) -> (Z, n, n), scale 1/(2P) (radon.py:145-160)."""
    filt = ramp_filter_apply(np.asarray(sino, dtype=np.float64))
    return np.stack([back_project_rows(p, s) for s in filt]) / (2.0 * sino.shape[1])


# ---------------------------------------------------------------- toeplitz
# toeplitz.py:46-241

_BATCH_BYTES = 64 * 2 ** 20


def padded_side_for(n: int) -> int:
    """Smallest odd 7-smooth >= 2n-1 (toeplitz.py:53-60)."""
    v = 2 * n - 1
    v += 1 - v % 2

    def smooth(x):
        for f in (2, 3, 5, 7):
            while x % f == 0:
                x //= f
        return x == 1

    while not smooth(v):
        v += 2
    return v


@dataclass
class Psf:
    m: int
    n: int
    nd: int
    main: np.ndarray
    flip: np.ndarray | None
    kernel: np.ndarray  # centred lag kernel K on the odd grid (for tests)


def build_psf(angles: np.ndarray, nd: int, n: int, tol: float = 1e-6, sigma: float = 2.0) -> Psf:
    """compute_psf on the odd padded grid (toeplitz.py:85-131)."""
    m = padded_side_for(n)
    p = make_plan(m, angles, nd, tol, sigma)
    k = type1(p, np.ones(p.samples.shape[0])).real
    spec = np.fft.fft2(np.fft.ifftshift(k))
    s = (m - n) // 2
    nyq = nyquist_mask(np.asarray(angles).size, nd)
    if nyq.any():
        kn = type1(p, np.where(nyq, 0.5, 0.0)).real
        sn = np.fft.fft2(np.fft.ifftshift(kn))
        ph = np.exp(-2j * np.pi * np.arange(m) * (2 * s + n - 1) / m)
        return Psf(m, n, nd, (spec - sn) / nd, -np.outer(ph, ph) * sn / nd, k)
    return Psf(m, n, nd, spec / nd, None, k)


def apply_batch(psf: Psf, batch: np.ndarray) -> np.ndarray:
    """R*R on a (Z, n, n) stack by padded FFT convolution (toeplitz.py:134-149)."""
    n, m = psf.n, psf.m
    s = (m - n) // 2
    batch = np.asarray(batch, dtype=np.float64)
    out = np.empty_like(batch)
    step = max(1, _BATCH_BYTES // (16 * m * m))
    for lo in range(0, batch.shape[0], step):
        hi = min(lo + step, batch.shape[0])
        pad = np.zeros((hi - lo, m, m), dtype=np.complex128)
        pad[:, s:s + n, s:s + n] = batch[lo:hi]
        F = np.fft.fft2(pad, axes=(1, 2))
        acc = F * psf.main[None]
        if psf.flip is not None:
            acc += np.conj(F) * psf.flip[None]
        out[lo:hi] = np.fft.ifft2(acc, axes=(1, 2)).real[:, s:s + n, s:s + n]
    return out


def apply_batch_threaded(psf: Psf, batch: np.ndarray, threads: int) -> np.ndarray:
    """Slice-parallel apply (numpy's FFT releases the GIL); the CPU baseline."""
    out = np.empty_like(np.asarray(batch, dtype=np.float64))

    def one(z):
        out[z] = apply_batch(psf, batch[z:z + 1])[0]

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, range(batch.shape[0])))
    return out


def rstar(p: Plan, sino: np.ndarray) -> np.ndarray:
    """R*g per slice (toeplitz.py:205)."""
    return np.stack([back_project_rows(p, s) for s in np.asarray(sino, dtype=np.float64)])


def fidelity_grad(psf: Psf, rs: np.ndarray, f: np.ndarray) -> np.ndarray:
    """toeplitz.py:233-241"""
    return apply_batch(psf, f) - rs


def fidelity_loss(psf: Psf, rs: np.ndarray, g_sq: float, f: np.ndarray) -> float:
    """toeplitz.py:226-230"""
    kf = apply_batch(psf, f)
    return float(0.5 * np.sum(f * kf) - np.sum(f * rs) + 0.5 * g_sq)


# ------------------------------------------------------------------ qggmrf
# qggmrf.py:43-217


@dataclass(frozen=True)
class Prior:
    sigma: float
    lam: float = 0.0
    p: float = 2.0
    q: float = 1.2
    T: float = 1.0


def stencil(three_d: bool):
    """Offsets (dz, dy, dx) in reference order and 1/dist weights (qggmrf.py:86-97)."""
    zs = (-1, 0, 1) if three_d else (0,)
    offs = [(a, b, c) for a in zs for b in (-1, 0, 1) for c in (-1, 0, 1) if (a, b, c) != (0, 0, 0)]
    inv = np.array([1.0 / math.sqrt(a * a + b * b + c * c) for a, b, c in offs])
    return offs, inv / inv.sum()


def half_stencil(three_d: bool):
    offs, w = stencil(three_d)
    return [(o, b) for o, b in zip(offs, w) if o > (0, 0, 0)]


def rho(pr: Prior, d):
    """qggmrf.py:117-121"""
    a = np.abs(np.asarray(d, dtype=np.float64))
    v = (a / (pr.T * pr.sigma)) ** (pr.p - pr.q)
    return a ** pr.p / (pr.p * pr.sigma ** pr.p) / (1.0 + v)


def rho_prime(pr: Prior, d):
    """qggmrf.py:124-130"""
    d = np.asarray(d, dtype=np.float64)
    a = np.abs(d)
    v = (a / (pr.T * pr.sigma)) ** (pr.p - pr.q)
    return np.sign(d) * a ** (pr.p - 1.0) / pr.sigma ** pr.p * (1.0 + pr.q / pr.p * v) / (1.0 + v) ** 2


def prior_grad(pr: Prior, vol: np.ndarray, halo_lo=None, halo_hi=None, three_d=None) -> np.ndarray:
    """sum_s b_s rho'(f_v - f_{v+s}) over in-range (or halo) neighbours (qggmrf.py:142-189)."""
    vol = np.asarray(vol, dtype=np.float64)
    z, h, w = vol.shape
    if three_d is None:
        three_d = z > 1
    offs, wts = stencil(three_d)
    ext = np.zeros((z + 2, h, w))
    ok = np.zeros(z + 2, dtype=bool)
    ext[1:-1], ok[1:-1] = vol, True
    if halo_lo is not None:
        ext[0], ok[0] = halo_lo, True
    if halo_hi is not None:
        ext[-1], ok[-1] = halo_hi, True
    g = np.zeros_like(vol)
    for (dz, dy, dx), b in zip(offs, wts):
        zok = ok[1 + dz:1 + dz + z].astype(np.float64)[:, None, None]
        ys, yn = slice(max(0, -dy), h - max(0, dy)), slice(max(0, dy), h + min(0, dy))
        xs, xn = slice(max(0, -dx), w - max(0, dx)), slice(max(0, dx), w + min(0, dx))
        nb = ext[1 + dz:1 + dz + z][:, yn, xn]
        g[:, ys, xs] += b * rho_prime(pr, vol[:, ys, xs] - nb) * zok
    return g


def prior_energy(pr: Prior, vol: np.ndarray, halo_hi=None, three_d=None) -> float:
    """Unordered-pair energy; +pairs into halo_hi (qggmrf.py:192-217)."""
    vol = np.asarray(vol, dtype=np.float64)
    z, h, w = vol.shape
    if three_d is None:
        three_d = z > 1
    tot = 0.0
    for (dz, dy, dx), b in half_stencil(three_d):
        ys, yn = slice(max(0, -dy), h - max(0, dy)), slice(max(0, dy), h + min(0, dy))
        xs, xn = slice(max(0, -dx), w - max(0, dx)), slice(max(0, dx), w + min(0, dx))
        tot += b * float(np.sum(rho(pr, vol[0:z - dz, ys, xs] - vol[dz:z, yn, xn])))
        if dz == 1 and halo_hi is not None:
            tot += b * float(np.sum(rho(pr, vol[z - 1, ys, xs] - halo_hi[yn, xn])))
    return tot


# ------------------------------------------------------------------ solver
# solver.py:67-180


def estimate_lipschitz(psf: Psf, pr: Prior) -> float:
    """Power iteration from default_rng(0x10E5) (solver.py:67-92)."""
    v = np.random.default_rng(0x10E5).standard_normal((psf.n, psf.n))
    nv = np.linalg.norm(v)
    est = 0.0
    for _ in range(30):
        w = apply_batch(psf, v[None])[0]
        nw = np.linalg.norm(w)
        if nw == 0.0:
            raise ValueError("power iteration on a zero operator")
        new = nw / nv
        v, nv = w / nw, 1.0
        if est > 0 and abs(new - est) < 1e-3 * new:
            est = new
            break
        est = new
    return 1.05 * (est + pr.lam * 2.0 / pr.sigma ** pr.p)


@dataclass(frozen=True)
class Record:
    iter: int
    objective: float
    fidelity: float
    prior: float
    grad_norm: float
    restarted: bool


def objective(psf, rs, g_sq, pr: Prior, f):
    """solver.py:95-101"""
    f = np.asarray(f, dtype=np.float64)
    kf = apply_batch(psf, f)
    fid = float(0.5 * np.sum(f * kf) - np.sum(f * rs) + 0.5 * g_sq)
    e = prior_energy(pr, f) if pr.lam != 0.0 else 0.0
    return fid + pr.lam * e, fid, e


def solve(psf, rs, g_sq, pr: Prior, f0, max_iters: int, L: float, tol: float = 1e-5,
          restart: bool = True, nonneg: bool = False, snapshots=None):
    """Momentum GD with function-value restart (solver.py:112-180)."""
    f = np.array(f0, dtype=np.float64)
    y = f
    t = 1.0
    three_d = f.shape[0] > 1
    obj, fid, e = objective(psf, rs, g_sq, pr, f)
    recs = []
    for k in range(1, max_iters + 1):
        grad = apply_batch(psf, y) - rs
        if pr.lam != 0.0:
            grad = grad + pr.lam * prior_grad(pr, y, three_d=three_d)
        gn = float(np.linalg.norm(grad))
        if k == 1:
            recs.append(Record(0, obj, fid, e, gn, False))
        fn = y - grad / L
        if nonneg:
            fn = np.maximum(fn, 0.0)
        on, fdn, en = objective(psf, rs, g_sq, pr, fn)
        if not np.isfinite(on):
            raise FloatingPointError(f"objective became non-finite at iteration {k}")
        rst = bool(restart and on > obj)
        if rst:
            tn, y = 1.0, fn
        else:
            tn = (1.0 + math.sqrt(1.0 + 4.0 * t * t)) / 2.0
            y = fn + ((t - 1.0) / tn) * (fn - f)
        recs.append(Record(k, on, fdn, en, gn, rst))
        if snapshots is not None:
            snapshots.append(fn.copy())
        done = (not rst) and abs(on - obj) <= tol * abs(obj)
        f, t, obj = fn, tn, on
        if done:
            break
    return f, recs


# ---------------------------------------------------------------- multires
# multires.py:93-242


def strided_indices(count: int, factor: int) -> np.ndarray:
    """multires.py:93-98"""
    red = -(-count // factor)
    start = max(0, ((count - 1) - factor * (red - 1)) // 2)
    return np.arange(start, count, factor)


def downsample_sinogram(angles, data, factor: int, downsample_angles: bool = False):
    """multires.py:101-125 -> (angles, data)"""
    data = np.asarray(data, dtype=np.float64)
    if factor == 1:
        return np.asarray(angles), data
    out = data[:, :, strided_indices(data.shape[2], factor)] / factor
    if downsample_angles:
        keep = np.arange(0, len(angles), factor)
        angles = np.asarray(angles)[keep]
        out = out[:, keep, :]
    if data.shape[0] > 1:
        out = out[strided_indices(data.shape[0], factor)]
    return np.asarray(angles), out


def lanczos(x, a: int = 3):
    """multires.py:128-142"""
    x = np.asarray(x, dtype=np.float64)
    ax = np.abs(x)
    inside = ax < a
    s = np.where(inside & (ax > 0), x, 1.0)
    v = a * np.sin(np.pi * s) * np.sin(np.pi * s / a) / (np.pi * s) ** 2
    v = np.where(ax == np.round(ax), 0.0, v)
    v = np.where(ax == 0, 1.0, v)
    return np.where(inside, v, 0.0)


def lanczos_matrix(n_src: int, n_tgt: int, a: int = 3) -> np.ndarray:
    """Edge-clamped, row-normalised interpolation matrix (multires.py:145-164)."""
    ratio = n_src / n_tgt
    cs, ct = (n_src - 1) / 2.0, (n_tgt - 1) / 2.0
    mat = np.zeros((n_tgt, n_src))
    for r in range(n_tgt):
        x = cs + (r - ct) * ratio
        taps = np.arange(int(math.ceil(x - a)), int(math.floor(x + a)) + 1)
        w = lanczos(x - taps, a)
        nz = w != 0.0
        np.add.at(mat[r], np.clip(taps[nz], 0, n_src - 1), w[nz])
        mat[r] /= mat[r].sum()
    return mat


def upsample(img: np.ndarray, side: int, slices: int | None = None) -> np.ndarray:
    """Separable z, y, x Lanczos-3 (multires.py:167-195)."""
    img = np.asarray(img, dtype=np.float64)
    m = lanczos_matrix(img.shape[-1], side)
    if img.ndim == 2:
        return m @ img @ m.T
    if slices is None:
        slices = int(round(img.shape[0] * side / img.shape[-1]))
    mz = lanczos_matrix(img.shape[0], slices)
    out = np.einsum("zi,iyx->zyx", mz, img)
    out = np.einsum("yi,ziw->zyw", m, out)
    return np.einsum("xi,zyi->zyx", m, out)


def solve_hierarchical(angles, sino, levels, iters, pr: Prior, L=None, use_fbp_init=False,
                       tol=1e-300, restart=True, downsample_angles=False):
    """Coarse-to-fine driver (multires.py:198-242); returns (estimate, records per level)."""
    n_levels = len(levels)
    est = None
    all_recs = []
    for lvl, side in enumerate(levels):
        fac = 1 << (n_levels - 1 - lvl)
        ang_l, sino_l = downsample_sinogram(angles, sino, fac, downsample_angles)
        nd = sino_l.shape[2]
        plan = make_plan(side, ang_l, nd)
        psf = build_psf(ang_l, nd, side)
        rs = rstar(plan, sino_l)
        g_sq = float(np.sum(sino_l ** 2))
        if est is None:
            f0 = fbp(plan, sino_l) if use_fbp_init else np.zeros((sino_l.shape[0], side, side))
        else:
            f0 = upsample(est, side, sino_l.shape[0]) if sino_l.shape[0] > 1 else \
                upsample(est[0], side)[None]
        Ll = L if L is not None else estimate_lipschitz(psf, pr)
        est, recs = solve(psf, rs, g_sq, pr, f0, iters[lvl], Ll, tol=tol, restart=restart)
        all_recs.append(recs)
    return est, all_recs


# ----------------------------------------------------------------- runtime
# runtime.py:108-125


def partition(n_slices: int, n_workers: int):
    """Balanced contiguous slabs, larger first: list of (begin, end)."""
    if n_workers < 1:
        raise ValueError("need at least one worker")
    if n_slices < n_workers:
        raise ValueError("more workers than slices")
    base, extra = divmod(n_slices, n_workers)
    out, b = [], 0
    for w in range(n_workers):
        s = base + (1 if w < extra else 0)
        out.append((b, b + s))
        b += s
    return out
