"""Adjoint NUFFT (type 1) on B200: Kaiser-Bessel gridding onto an oversampled grid.

Drop-in for the parts of tomoforge/nufft.py on the reconstruction path:
``NufftPlan`` / ``plan`` (nufft.py:104-176), ``type1`` (:203-223),
``kernel_width_for_tolerance`` (:54-57) and ``kaiser_bessel_fourier``
(:90-101).  The forward transform ``type2`` (data synthesis)
runs on the same tables through ``type2_stack`` (csrc/nufft.cu, k_interp).

The plan keeps the reference's kernel width and shape parameter; its device
tables are built once per (plan, device) on the host in float64:

* the GPU grid side ``gpu_side`` = the smallest power of two >= max(32,
  reference ``os_side``) -- equal to the reference grid at sigma = 2 and
  power-of-two N, finer otherwise (never less accurate);
* per sample: the first window index on both axes and the 2w Kaiser-Bessel
  weights, evaluated exactly (the reference interpolates a 16384/unit table);
* the samples binned into 32 x 32 grid tiles (CSR, sample order kept), which
  makes the atomic-free spreading kernel deterministic;
* deapodisation 1/KB^(x'/os) on the N output pixels (same clamp as the
  reference) and the centring pre-phase e^{-2 pi i a (N//2) / os} per grid index.
"""

from __future__ import annotations

import collections
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .geometry import ImageGrid, PolarSampling

__all__ = [
    "SpreadKernel",
    "NufftPlan",
    "plan",
    "type1",
    "type2",
    "direct_dft",
    "kernel_width_for_tolerance",
    "kaiser_bessel_fourier",
]

_MIN_TOLERANCE = 1e-14
_MAX_TOLERANCE = 1e-1
_BETA_SCALE = {3: 0.94, 4: 0.96, 5: 0.97, 6: 0.98, 7: 0.985}
_BETA_SCALE_DEFAULT = 0.99
TILE = 32  # grid tile side of the spreading kernel (csrc/nufft.cu, k_spread)
BAND = 4  # grid rows per warp of k_spread: the CSR lists samples per (tile, band)
BANDS = TILE // BAND


def kernel_width_for_tolerance(tolerance: float) -> int:
    """w = ceil(log10(1/eps)) + 1, at least 2 (nufft.py:54-57)."""
    digits = -np.log10(tolerance)
    return max(2, int(np.ceil(digits - 1e-9)) + 1)


def kaiser_bessel_fourier(xi, width: int, beta: float) -> np.ndarray:
    """Fourier transform of the KB kernel at xi cycles/grid unit (nufft.py:90-101)."""
    z = beta * beta - (np.pi * width * np.asarray(xi, dtype=np.float64)) ** 2
    sq = np.sqrt(np.abs(z))
    with np.errstate(invalid="ignore", divide="ignore"):
        out = np.where(z > 0.0, np.sinh(sq) / np.where(sq == 0, 1.0, sq), np.sinc(sq / np.pi))
    out = np.where(sq == 0.0, 1.0, out)
    return width * out


def _kb(x: np.ndarray, width: int, beta: float) -> np.ndarray:
    """I0(beta sqrt(1 - (2x/w)^2)) on |x| <= w/2, else 0 (nufft.py:80-87, exact)."""
    arg = 1.0 - (2.0 * np.asarray(x, dtype=np.float64) / width) ** 2
    return np.where(arg >= 0.0, np.i0(beta * np.sqrt(np.maximum(arg, 0.0))), 0.0)


TABLE_SAMPLES_PER_UNIT = 16384


@dataclass(frozen=True)
class SpreadKernel:
    """Tabulated Kaiser-Bessel kernel on |x| <= width/2 (nufft.py:60-87).

    Kept for API compatibility (``NufftPlan.kernel``); the GPU plan evaluates
    the same kernel exactly in fp64 (k_plan_weights) instead of interpolating."""

    width: int
    beta: float
    lookup: np.ndarray = field(repr=False)
    step: float

    def __call__(self, x: np.ndarray) -> np.ndarray:
        t = np.abs(x) / self.step
        idx = t.astype(np.int64)
        inside = idx < self.lookup.size - 1
        idx = np.where(inside, idx, 0)
        frac = t - idx
        vals = self.lookup[idx] * (1.0 - frac) + self.lookup[idx + 1] * frac
        return np.where(inside, vals, 0.0)


def _build_kernel(width: int, beta: float) -> SpreadKernel:
    """nufft.py:80-87"""
    n_tab = int(width / 2 * TABLE_SAMPLES_PER_UNIT) + 2
    step = (width / 2) / (n_tab - 2)
    x = np.arange(n_tab) * step
    table = _kb(x, width, beta)
    table.setflags(write=False)
    return SpreadKernel(width=width, beta=beta, lookup=table, step=step)


def gpu_grid_side(os_side: int) -> int:
    g = 32
    while g < os_side:
        g *= 2
    return g


class PlanTables:
    """Host (float64 -> fp32/int32 numpy) tables of one plan; see module docstring.

    ``weights=False`` skips the Kaiser-Bessel weights (the device builds them,
    csrc/nufft.cu k_plan_weights); the window starts, the tile CSR, the
    deapodisation and the pre-phase are always built here."""

    def __init__(self, n: int, samples: np.ndarray, width: int, beta: float, os_side: int,
                 weights: bool = True, csr: bool = True):
        g = gpu_grid_side(os_side)
        self.side, self.width, self.beta = n, width, beta
        self.grid = g
        kx, ky = samples[:, 0], samples[:, 1]

        def start(k):
            return np.ceil(k * g / (2.0 * np.pi) - width / 2.0).astype(np.int64)

        def kb_weights(k, st):
            eta = k * g / (2.0 * np.pi)
            idx = st[:, None] + np.arange(width)[None, :]
            return _kb(idx - eta[:, None], width, beta)

        sa, sb = start(kx), start(ky)
        a0, b0 = sa % g, sb % g
        self.ab = np.stack([a0, b0], axis=1).astype(np.int32)
        self.wts = None
        if weights:
            self.wts = np.concatenate([kb_weights(kx, sa), kb_weights(ky, sb)],
                                      axis=1).astype(np.float32)
        xprime = np.arange(n) - n // 2
        dk = kaiser_bessel_fourier(xprime / g, width, beta)
        floor = 1e-12 * np.max(np.abs(dk))
        dk = np.where(np.abs(dk) < floor, floor, dk)
        self.deapod = (1.0 / dk).astype(np.float32)
        # output pixel ix sits at grid offset ix - N//2: shift it to ix (first N outputs)
        self.prephase = np.exp(-2j * np.pi * np.arange(g) * (n // 2) / g).astype(np.complex64)
        self.tile_ptr = self.tile_idx = None
        if csr:
            self.tile_ptr, self.tile_idx = self._bin(a0, b0, g, width)

    @staticmethod
    def _bin(a0, b0, g, width):
        """CSR of the samples whose window touches each 4-row band of each 32 x 32
        tile (entry tile * 8 + band, tile = tb * (g/32) + ta), samples ascending:
        warp `band` of the tile's CTA walks only its own list."""
        nt = g // TILE
        m = np.arange(a0.size, dtype=np.int64)
        ta = [a0 // TILE, ((a0 + width - 1) % g) // TILE]
        rows = (b0[:, None] + np.arange(width)[None, :]) % g
        bands = rows // BAND  # global band of each window row, (S, W)
        first = np.ones_like(bands, dtype=bool)
        first[:, 1:] = bands[:, 1:] != bands[:, :-1]  # each touched band once
        keys, ids = [], []
        for i, xa in enumerate(ta):
            keep_a = np.ones(a0.size, bool) if i == 0 else xa != ta[0]
            sel = first & keep_a[:, None]
            gb = bands[sel]
            tb, w = gb // BANDS, gb % BANDS
            keys.append(((tb * nt + np.broadcast_to(xa[:, None], bands.shape)[sel]) * BANDS + w))
            ids.append(np.broadcast_to(m[:, None], bands.shape)[sel])
        keys = np.concatenate(keys)
        ids = np.concatenate(ids)
        order = np.lexsort((ids, keys))  # by (tile, band), then sample index
        keys, ids = keys[order], ids[order]
        ptr = np.searchsorted(keys, np.arange(nt * nt * BANDS + 1)).astype(np.int32)
        return ptr, ids.astype(np.int32)


def _band_csr_device(ab: torch.Tensor, g: int, width: int):
    """PlanTables._bin on the device (torch stable sort; bit-identical CSR): the
    samples whose window touches each (tile, 4-row band), in sample order."""
    nt = g // TILE
    a0, b0 = ab[:, 0].long(), ab[:, 1].long()
    s = a0.numel()
    ta0 = a0 // TILE
    ta1 = ((a0 + width - 1) % g) // TILE
    rows = (b0[:, None] + torch.arange(width, device=ab.device)) % g
    bands = rows // BAND
    first = torch.ones_like(bands, dtype=torch.bool)
    first[:, 1:] = bands[:, 1:] != bands[:, :-1]
    tb, w = bands // BANDS, bands % BANDS
    k0 = torch.where(first, (tb * nt + ta0[:, None]) * BANDS + w, -1)
    k1 = torch.where(first & (ta1 != ta0)[:, None], (tb * nt + ta1[:, None]) * BANDS + w, -1)
    keys = torch.stack([k0, k1], dim=1).reshape(-1)  # sample-major: stable sort keeps order
    ids = torch.arange(s, device=ab.device, dtype=torch.int32).repeat_interleave(2 * width)
    ok = keys >= 0
    keys, ids = keys[ok], ids[ok]
    keys, order = torch.sort(keys, stable=True)
    ptr = torch.searchsorted(keys, torch.arange(nt * nt * BANDS + 1, device=ab.device))
    return ptr.to(torch.int32), ids[order].contiguous()


def _tile_order_device(tile_ptr: torch.Tensor) -> torch.Tensor:
    """Launch order of the spreading tiles: by descending band-list work (stable),
    so the dense centre tiles start first instead of trailing the launch."""
    ptr = tile_ptr.long().reshape(-1)
    work = (ptr[BANDS::BANDS] - ptr[:-1:BANDS])  # samples visited per tile, all bands
    return torch.sort(-work, stable=True)[1].to(torch.int32).contiguous()


_TABLE_CACHE: "collections.OrderedDict[tuple, dict]" = collections.OrderedDict()
_TABLE_CACHE_SIZE = 8


def _shared_device_tables(key: tuple) -> dict:
    """Per-geometry dict {device index: tables}, least-recently-used, 8 geometries."""
    d = _TABLE_CACHE.get(key)
    if d is None:
        d = _TABLE_CACHE[key] = {}
        while len(_TABLE_CACHE) > _TABLE_CACHE_SIZE:
            _TABLE_CACHE.popitem(last=False)
    else:
        _TABLE_CACHE.move_to_end(key)
    return d


class NufftPlan:
    """Reusable type-1 plan for (grid side, polar sampling, tolerance) (nufft.py:104-168)."""

    def __init__(self, grid_side: int, sampling: PolarSampling, tolerance: float,
                 oversampling: float = 2.0):
        if not (_MIN_TOLERANCE < tolerance < _MAX_TOLERANCE):
            raise ValueError(
                f"tolerance must lie in ({_MIN_TOLERANCE:g}, {_MAX_TOLERANCE:g}), got {tolerance:g}"
            )
        if oversampling < 1.25:
            raise ValueError("oversampling factor must be >= 1.25")
        if grid_side < 2:
            raise ValueError("grid side must be at least 2")
        self.grid_side = int(grid_side)
        self.sampling = sampling
        self.tolerance = float(tolerance)
        self.oversampling = float(oversampling)
        self.kernel_width = kernel_width_for_tolerance(tolerance)
        gamma = _BETA_SCALE.get(self.kernel_width, _BETA_SCALE_DEFAULT)
        self.kernel_params = gamma * np.pi * self.kernel_width * (1.0 - 1.0 / (2.0 * oversampling))
        self._kernel = None
        os_side = int(np.ceil(oversampling * self.grid_side))
        if os_side % 2:
            os_side += 1
        self.os_side = os_side
        self.gpu_side = gpu_grid_side(os_side)
        if self.gpu_side > 8192:
            raise NotImplementedError(f"oversampled grid {self.gpu_side} exceeds 8192")
        n = self.grid_side
        delta = n // 2 - (n - 1) / 2.0
        kx, ky = sampling.samples[:, 0], sampling.samples[:, 1]
        self._phase = np.exp(-1j * (kx + ky) * delta)
        self._tables = None
        # device tables are shared by plans of the same geometry (repeated
        # reconstructions, the per-level plans of solve_hierarchical)
        self._device_tables = _shared_device_tables(
            (self.grid_side, self.kernel_width, float(self.kernel_params), self.os_side,
             sampling.radial_count, np.asarray(sampling.angles, dtype=np.float64).tobytes()))

    @property
    def sample_count(self) -> int:
        return self.sampling.count

    @property
    def kernel(self) -> SpreadKernel:
        """The reference's tabulated spreading kernel (built on first use)."""
        if self._kernel is None:
            self._kernel = _build_kernel(self.kernel_width, self.kernel_params)
        return self._kernel

    @property
    def tables(self) -> PlanTables:
        """Host tables including the Kaiser-Bessel weights (numpy, float64 math)."""
        if self._tables is None:
            self._tables = PlanTables(self.grid_side, np.asarray(self.sampling.samples),
                                      self.kernel_width, self.kernel_params, self.os_side)
        return self._tables

    def device_tables(self) -> dict:
        """fp32/int32 tables on the current CUDA device (built once per device): the
        window starts and Kaiser-Bessel weights by k_plan_weights (fp64 on the GPU),
        the tile CSR / deapodisation / pre-phase from the host."""
        dev = _lib.device()
        t = self._device_tables.get(dev.index)
        if t is None:
            lib = _lib.ensure_ready()
            samples = np.ascontiguousarray(self.sampling.samples, dtype=np.float64)
            h = self._tables or PlanTables(self.grid_side, samples, self.kernel_width,
                                           self.kernel_params, self.os_side, weights=False,
                                           csr=False)
            up = lambda a: torch.from_numpy(np.array(a, copy=True, order="C")).to(dev)  # noqa: E731
            kxy = up(samples)
            ab = torch.empty((samples.shape[0], 2), dtype=torch.int32, device=dev)
            wts = torch.empty((samples.shape[0], 2 * self.kernel_width), dtype=torch.float32,
                              device=dev)
            _lib.check(lib.tf_nufft_plan_weights(kxy.data_ptr(), samples.shape[0], self.gpu_side,
                                                 self.kernel_width, float(self.kernel_params),
                                                 ab.data_ptr(), wts.data_ptr(),
                                                 _lib.stream_handle()), "tf_nufft_plan_weights")
            # the tile CSR was binned from the host window starts: they must agree
            if not np.array_equal(ab.cpu().numpy(), h.ab):
                raise RuntimeError("NUFFT plan: device window starts differ from the host binning")
            t = {
                "ab": ab, "wts": wts, "deapod": up(h.deapod),
                "prephase": up(h.prephase.view(np.float32)),
                **dict(zip(("tile_ptr", "tile_idx"), _band_csr_device(ab, self.gpu_side,
                                                                       self.kernel_width))),
                "tile_order": None,
                "sphase": None,
            }
            self._device_tables[dev.index] = t
        return t

    def detector_sample_phase(self) -> torch.Tensor:
        """Per-sample factor e^{i w_j [(Nd-1)/2 + delta (cos t + sin t)]} / Nd on the device.

        Folds the detector-centring phase and 1/Nd of radon._back_project_rows
        (radon.py:124-128) with conj(plan phase) of type1 (nufft.py:213)."""
        t = self.device_tables()
        if t["sphase"] is None:
            nd = self.sampling.radial_count
            w = np.repeat(self.sampling.radial_freqs[None], self.sampling.angles.size, 0).ravel()
            ph = np.exp(1j * w * (nd - 1) / 2.0) / nd * np.conj(self._phase)
            t["sphase"] = torch.from_numpy(ph.astype(np.complex64).view(np.float32)).to(
                _lib.device())
        return t["sphase"]


    def sample_factor(self, kind: str) -> torch.Tensor:
        """Per-sample complex64 factor on the device: ``"type2"`` = the plan phase
        e^{-i (kx+ky) delta} (nufft.py:199); ``"project"`` = that times the detector
        phase e^{-i w_j (Nd-1)/2} (radon.py:90)."""
        t = self.device_tables()
        key = "f_" + kind
        if t.get(key) is None:
            ph = self._phase
            if kind == "project":
                nd = self.sampling.radial_count
                w = np.repeat(self.sampling.radial_freqs[None], self.sampling.angles.size,
                              0).ravel()
                ph = ph * np.exp(-1j * w * (nd - 1) / 2.0)
            t[key] = torch.from_numpy(ph.astype(np.complex64).view(np.float32)).to(_lib.device())
        return t[key]


def plan(grid_side: int, sampling: PolarSampling, tolerance: float,
         oversampling: float = 2.0) -> NufftPlan:
    """nufft.py:171-176"""
    return NufftPlan(grid_side, sampling, tolerance, oversampling)


# spreading workspace per launch: ~10 slices of a 4096^2 oversampled grid; fewer
# slices per launch leave a tail of dense centre tiles (R*g on 64 x 2048^2:
# 11.2 ms at 5 slices, 9.3 ms at 10 with the heaviest-first tile order)
_WS_BYTES = 2 << 30


def type1_stack(p: NufftPlan, samples: torch.Tensor, out: torch.Tensor | None = None,
                scale: float = 1.0, complex_out: bool = False) -> torch.Tensor:
    """Spread + inverse FFT + deapodise a (Z, S) complex64 device stack of samples
    (already multiplied by conj(phase)); returns (Z, N, N) fp32 (real part) or
    complex64."""
    lib = _lib.ensure_ready()
    t = p.device_tables()
    n, g = p.grid_side, p.gpu_side
    if samples.dtype != torch.complex64 or not samples.is_contiguous() or samples.dim() != 2:
        raise ValueError("samples must be a contiguous (Z, S) complex64 device tensor")
    z = samples.shape[0]
    if samples.shape[1] != p.sample_count:
        raise ValueError(f"expected {p.sample_count} samples, got {samples.shape[1]}")
    if out is None:
        out = torch.empty((z, n, n), dtype=torch.complex64 if complex_out else torch.float32,
                          device=samples.device)
    per = lib.tf_nufft_workspace_bytes(g, 1)
    chunk = max(1, min(z, _WS_BYTES // per))
    ws = _device.workspace(per * chunk, tag="nufft")
    if t.get("tile_order") is None:
        t["tile_order"] = _tile_order_device(t["tile_ptr"])
    _lib.check(lib.tf_nufft_type1(
        samples.data_ptr(), samples.shape[1], z, n, g, p.kernel_width, t["tile_ptr"].data_ptr(),
        t["tile_idx"].data_ptr(), t["tile_order"].data_ptr(), t["ab"].data_ptr(),
        t["wts"].data_ptr(),
        t["prephase"].data_ptr(), t["deapod"].data_ptr(), float(scale), int(complex_out),
        out.data_ptr(), ws.data_ptr(), per * chunk, _lib.stream_handle()), "tf_nufft_type1")
    return out


def type1(p: NufftPlan, samples) -> np.ndarray:
    """Polar samples -> complex (N, N) grid, adjoint of type2 (nufft.py:203-223)."""
    samples = np.asarray(samples, dtype=np.complex128)
    if samples.shape != (p.sample_count,):
        raise ValueError(f"expected {p.sample_count} samples, got shape {samples.shape}")
    c = (samples * np.conj(p._phase)).astype(np.complex64)
    d = torch.from_numpy(c[None]).to(_lib.device())
    out = type1_stack(p, d, complex_out=True)
    return out[0].cpu().numpy().astype(np.complex128)



def type2_stack(p: NufftPlan, images: torch.Tensor, factor: str = "type2") -> torch.Tensor:
    """(Z, N, N) fp32 device images -> (Z, S) complex64 samples (type2 x factor)."""
    lib = _lib.ensure_ready()
    t = p.device_tables()
    n, g = p.grid_side, p.gpu_side
    if images.dim() != 3 or tuple(images.shape[1:]) != (n, n):
        raise ValueError(f"image shape {tuple(images.shape[1:])} does not match plan grid {n}x{n}")
    x = images.to(torch.float32).contiguous()
    z = x.shape[0]
    out = torch.empty((z, p.sample_count), dtype=torch.complex64, device=x.device)
    per = lib.tf_nufft_type2_workspace_bytes(n, g, 1)
    chunk = max(1, min(z, _WS_BYTES // per))
    ws = _device.workspace(per * chunk, tag="nufft2")
    fac = p.sample_factor(factor)
    _lib.check(lib.tf_nufft_type2(
        x.data_ptr(), z, n, g, p.kernel_width, t["ab"].data_ptr(), t["wts"].data_ptr(),
        t["prephase"].data_ptr(), t["deapod"].data_ptr(), fac.data_ptr(), p.sample_count,
        out.data_ptr(), ws.data_ptr(), per * chunk, _lib.stream_handle()), "tf_nufft_type2")
    return out


def type2(p: NufftPlan, image) -> np.ndarray:
    """Grid -> polar samples c_m = sum_n f[n] exp(-i k_m . x_n) (nufft.py:184-200)."""
    arr = image.data if isinstance(image, ImageGrid) else np.asarray(image)
    n = p.grid_side
    if arr.shape != (n, n):
        raise ValueError(f"image shape {arr.shape} does not match plan grid {n}x{n}")
    out = type2_stack(p, _device.to_device(np.asarray(arr, dtype=np.float64)[None]))
    return out[0].cpu().numpy().astype(np.complex128)


_DIRECT_MAX_SIDE = 128


def direct_dft(sampling: PolarSampling, image) -> np.ndarray:
    """Brute-force type-2 sum in fp64 on the GPU; the reference's accuracy oracle for
    N <= 128 (nufft.py:230-249)."""
    arr = image.data if isinstance(image, ImageGrid) else np.asarray(image)
    n = arr.shape[0]
    if arr.shape != (n, n):
        raise ValueError("direct_dft needs a square image")
    if n > _DIRECT_MAX_SIDE:
        raise ValueError(f"direct_dft is an oracle for N <= {_DIRECT_MAX_SIDE}, got N={n}")
    lib = _lib.ensure_ready()
    dev = _lib.device()
    img = torch.from_numpy(np.array(arr, dtype=np.float64, order="C")).to(dev)
    kxy = torch.from_numpy(np.array(sampling.samples, dtype=np.float64, order="C")).to(dev)
    out = torch.empty((sampling.count, 2), dtype=torch.float64, device=dev)
    _lib.check(lib.tf_direct_dft(img.data_ptr(), n, kxy.data_ptr(), sampling.count,
                                 out.data_ptr(), _lib.stream_handle()), "tf_direct_dft")
    o = out.cpu().numpy()
    return o[:, 0] + 1j * o[:, 1]
