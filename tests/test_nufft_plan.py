"""CPU checks of the NUFFT plan tables and the kernels' index algebra.

The CUDA kernels of csrc/nufft.cu consume host-built tables (window starts,
Kaiser-Bessel weights, tile CSR, deapodisation, pre-phase).  These tests replay
the kernels' arithmetic in numpy on those same tables and compare with the
oracle (pinned to the reference by tests/test_oracle.py), so the conventions
are verified without a GPU.
"""

import numpy as np
import pytest

import oracle as O
from conftest import golden, rel_l2
from paper_2603_28756_b200.geometry import ScanGeometry, polar_sampling
from paper_2603_28756_b200.nufft import BAND, BANDS, TILE, NufftPlan


def _plan(n, n_ang, nd, tol=1e-6, sigma=2.0):
    ang = np.linspace(0, np.pi, n_ang, endpoint=False)
    geom = ScanGeometry(angles=ang, detector_bins=nd, image_side=n)
    return ang, NufftPlan(n, polar_sampling(geom), tol, sigma)


def emulate_type1(p: NufftPlan, c: np.ndarray) -> np.ndarray:
    """k_spread + k_nufft_rows + k_nufft_cols in numpy (complex output)."""
    t = p.tables
    g, w, n = t.grid, t.width, t.side
    grid = np.zeros((g, g), dtype=np.complex128)  # [b][a]
    a_idx = (t.ab[:, 0:1] + np.arange(w)[None]) % g
    b_idx = (t.ab[:, 1:2] + np.arange(w)[None]) % g
    wx, wy = t.wts[:, :w].astype(np.float64), t.wts[:, w:].astype(np.float64)
    vals = c[:, None, None] * wy[:, :, None] * wx[:, None, :]
    np.add.at(grid, (b_idx[:, :, None], a_idx[:, None, :]), vals)
    pre = t.prephase.astype(np.complex128)
    grid *= pre[:, None] * pre[None, :]
    # rows: inverse along a, keep first g/2 (ix); cols: inverse along b, keep iy < n
    h = np.fft.ifft(grid, axis=1)[:, : g // 2] * g
    out = (np.fft.ifft(h, axis=0)[:n] * g).T[:n, :n]  # [ix][iy]
    d = t.deapod.astype(np.float64)
    return out * np.outer(d, d)


@pytest.mark.parametrize("n,n_ang,nd", [(32, 20, 40), (24, 9, 48), (33, 10, 33), (64, 45, 64)])
def test_emulated_gridding_matches_oracle_type1(n, n_ang, nd):
    ang, p = _plan(n, n_ang, nd)
    rng = np.random.default_rng(n + nd)
    c = rng.standard_normal(p.sample_count) + 1j * rng.standard_normal(p.sample_count)
    ref = O.type1(O.make_plan(n, ang, nd), c)
    got = emulate_type1(p, c * np.conj(p._phase))
    assert rel_l2(got, ref) < 2e-6


def test_emulated_type1_matches_reference_fixture():
    d = golden("nufft_n32_p20_nd40.npz")
    geom = ScanGeometry(angles=d["angles"], detector_bins=40, image_side=32)
    p = NufftPlan(32, polar_sampling(geom), 1e-6)
    got = emulate_type1(p, d["c"] * np.conj(p._phase))
    assert rel_l2(got, d["type1"]) < 2e-6


def test_band_csr_covers_every_window():
    """k_spread's CSR: per (32 x 32 tile, 4-row band) the samples whose window
    touches it, in sample order (deterministic per-point accumulation order)."""
    _, p = _plan(48, 12, 64)
    t = p.tables
    g, w, nt = t.grid, t.width, t.grid // TILE
    ptr, idx = t.tile_ptr, t.tile_idx
    assert ptr.size == nt * nt * BANDS + 1
    assert ptr[0] == 0 and ptr[-1] == idx.size and np.all(np.diff(ptr) >= 0)
    cols = (t.ab[:, 0:1] + np.arange(w)) % g
    rows = (t.ab[:, 1:2] + np.arange(w)) % g
    for tile in range(nt * nt):
        ta, tb = tile % nt, tile // nt
        in_a = (cols // TILE == ta).any(1)
        for band in range(BANDS):
            members = idx[ptr[tile * BANDS + band]:ptr[tile * BANDS + band + 1]]
            assert np.all(np.diff(members) > 0)
            in_b = (rows // BAND == tb * BANDS + band).any(1)
            np.testing.assert_array_equal(members, np.nonzero(in_a & in_b)[0])


def _stockham(x, tw, L, r, nd):
    """smem_fft_pow2 on r interleaved sequences buf[s*L + n1]."""
    buf = x.copy()
    half = L // 2
    ls = 1
    while ls < L:
        tmp = np.empty_like(buf)
        for s in range(r):
            for j in range(half):
                k = j & (ls - 1)
                a = buf[s * L + j]
                b = buf[s * L + j + half] * tw[k * (nd // (2 * ls))]
                o = s * L + ((j - k) << 1) + k
                tmp[o], tmp[o + ls] = a + b, a - b
        buf = tmp
        ls *= 2
    return buf


def emulate_detector_dft(x, inverse=False):
    nd = x.size
    L = 1
    while nd % (2 * L) == 0:
        L *= 2
    r = nd // L
    tw = np.exp((2j if inverse else -2j) * np.pi * np.arange(nd) / nd)
    b = np.empty(nd, complex)
    for i in range(nd):
        b[(i % r) * L + i // r] = x[i]
    F = _stockham(b, tw, L, r, nd)
    out = np.empty(nd, complex)
    for k in range(nd):
        k1 = k & (L - 1)
        out[k] = sum(F[s * L + k1] * tw[(s * k) % nd] for s in range(r))
    return out


@pytest.mark.parametrize("nd", [1, 2, 8, 12, 33, 40, 64, 80, 96])
def test_detector_dft_algebra(nd):
    x = np.random.default_rng(nd).standard_normal(nd) + 0j
    np.testing.assert_allclose(emulate_detector_dft(x), np.fft.fft(x), atol=1e-10 * max(1, nd))
    np.testing.assert_allclose(emulate_detector_dft(x, True), np.fft.ifft(x) * nd,
                               atol=1e-10 * max(1, nd))


def test_plan_validation():
    ang = np.linspace(0, np.pi, 4, endpoint=False)
    s = polar_sampling(ScanGeometry(angles=ang, detector_bins=16, image_side=16))
    with pytest.raises(ValueError):
        NufftPlan(16, s, 1.0)
    with pytest.raises(ValueError):
        NufftPlan(16, s, 1e-6, oversampling=1.0)
    p = NufftPlan(16, s, 1e-6)
    assert p.kernel_width == 7 and p.os_side == 32 and p.gpu_side == 32
    assert NufftPlan(200, s, 1e-6).gpu_side == 512


def test_spread_kernel_table():
    """nufft.py:60-87: tabulated I0 kernel, exact at table nodes, zero off support."""
    _, p = _plan(16, 4, 16)
    k = p.kernel
    assert k.width == 7 and k(np.array([0.0]))[0] == pytest.approx(np.i0(p.kernel_params))
    assert k(np.array([3.6]))[0] == 0.0
    x = np.linspace(-3.4, 3.4, 41)
    beta, w = p.kernel_params, 7
    exact = np.i0(beta * np.sqrt(1 - (2 * x / w) ** 2))
    np.testing.assert_allclose(k(x), exact, rtol=1e-6)  # linear interpolation of the table


@pytest.mark.parametrize("n,n_ang,nd", [(48, 12, 64), (33, 10, 33)])
def test_band_csr_device_builder_matches_host(n, n_ang, nd):
    """device_tables builds the CSR with torch (here on the CPU): identical to _bin."""
    import torch

    from paper_2603_28756_b200.nufft import _band_csr_device

    _, p = _plan(n, n_ang, nd)
    t = p.tables
    ptr, idx = _band_csr_device(torch.from_numpy(t.ab), t.grid, t.width)
    np.testing.assert_array_equal(ptr.numpy(), t.tile_ptr)
    np.testing.assert_array_equal(idx.numpy(), t.tile_idx)
