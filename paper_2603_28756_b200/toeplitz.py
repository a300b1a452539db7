"""Normal-operator (Toeplitz) application and data-fidelity loss/gradient on B200.

Drop-in for tomoforge/toeplitz.py.  R*R acts on an N x N slice as a
convolution with a real, centro-symmetric lag kernel (toeplitz.py:1-19); for
even detector sizes an extra kernel acts on the flipped image.  The reference
synthesises the kernel with an adjoint NUFFT on an odd padded grid
(toeplitz.py:85-124); this build evaluates the same kernel in closed form on
the GPU (fp64 Dirichlet sums), re-embeds it on an even power-of-two grid
M >= 2N-1 and runs the fused real-FFT convolution of csrc/toeplitz.cu
(K1 rows -> K2 columns x PSF -> K3 rows).  See DESIGN.md §3 for the algebra.
"""

from __future__ import annotations

import collections
import functools
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .geometry import ImageGrid, PolarSampling, Sinogram, Volume

__all__ = [
    "PsfKernel",
    "FidelityContext",
    "padded_side_for",
    "fft_side_for",
    "compute_psf",
    "build_psf",
    "fidelity_context",
    "toeplitz_apply",
    "fidelity_loss",
    "fidelity_grad",
    "clear_caches",
]

# slices processed per apply pass; bounds the half-spectrum workspace
_MAX_CHUNK_BYTES = 4 << 30


def _is_7smooth(v: int) -> bool:
    for p in (2, 3, 5, 7):
        while v % p == 0:
            v //= p
    return v == 1


def padded_side_for(source_side: int) -> int:
    """Reference padding rule (toeplitz.py:53-60): smallest odd 7-smooth >= 2N-1."""
    v = 2 * source_side - 1
    v += 1 - v % 2
    while not _is_7smooth(v):
        v += 2
    return v


def fft_side_for(source_side: int) -> int:
    """FFT grid side used on the GPU: the smallest M >= 2N-1 that is a power of two
    or 5 * 2^k, k = 8..10 (radix-5 step: N = 640 / 1280 / 2560 -> 1280 / 2560 / 5120)."""
    m = _lib.load().tf_fft_side(int(source_side))
    if m < 0:
        _lib.check(m, "tf_fft_side")
    return m


@dataclass(frozen=True)
class PsfKernel:
    """Fourier-domain kernel of the projection normal operator (toeplitz.py:63-82).

    Reference fields keep their meaning: ``padded_side`` is the reference's odd
    7-smooth side m >= 2N-1 (``padded_side_for``), ``embed_offset`` = (m - N) // 2
    and ``spectrum`` the fp64 (m, m) fft2 of the ifftshifted lag kernel -- computed
    on first access (closed-form fp64 kernel on the device, fp64 FFT, read-only
    host array).  The apply path uses the device spectra on the even grid
    ``fft_side`` = M:

    ``pq``: (M/2+1, M, 2) fp32 = ((A + Re B)/M^2, (A - Re B)/M^2) with ``A`` the
    spectrum of (K - K_nyq)/Nd and ``B`` that of the flip kernel -K_nyq/Nd times
    the flip phase; ``bi``: (M/2+1, M) fp32 = Im B / M^2.  Rows are ky (half
    spectrum), columns kx.
    """

    padded_side: int
    source_side: int
    radial_count: int
    pq: torch.Tensor = field(repr=False)
    bi: torch.Tensor = field(repr=False)
    has_flip: bool = False
    fft_side: int = 0
    angles: np.ndarray = field(default=None, repr=False, compare=False, hash=False)

    @property
    def embed_offset(self) -> int:
        return (self.padded_side - self.source_side) // 2

    @property
    def device(self) -> torch.device:
        return self.pq.device

    @functools.cached_property
    def spectrum(self) -> np.ndarray:
        """fft2(ifftshift(K)) on the odd m x m grid, K(d) = sum_theta sum_j
        cos(w_j d.e_theta) (toeplitz.py:102-103); read-only complex128."""
        lib = _lib.ensure_ready()
        m = self.padded_side
        cs = np.stack([np.cos(self.angles), np.sin(self.angles)], axis=1)
        d_cs = torch.from_numpy(np.ascontiguousarray(cs, dtype=np.float64)).to(self.device)
        k = torch.empty((m, m), dtype=torch.float64, device=self.device)
        _lib.check(lib.tf_psf_kernel(m, int(self.angles.size), d_cs.data_ptr(),
                                     int(self.radial_count), k.data_ptr(), _lib.stream_handle()),
                   "tf_psf_kernel")
        spec = torch.fft.fft2(k).cpu().numpy()  # one-time fp64 library FFT (not the apply path)
        spec.setflags(write=False)
        return spec


def _check_tolerance(tolerance: float, oversampling: float) -> None:
    # same admissible ranges as the reference NUFFT plan (nufft.py:115-120);
    # the closed-form kernel itself is exact to fp64 rounding
    if not (1e-14 < tolerance < 1e-1):
        raise ValueError(f"tolerance must lie in (1e-14, 0.1), got {tolerance:g}")
    if oversampling < 1.25:
        raise ValueError("oversampling factor must be >= 1.25")


_PSF_CACHE: "collections.OrderedDict[tuple, PsfKernel]" = collections.OrderedDict()
_PSF_CACHE_SIZE = 4  # ~100 MB of spectra each at N = 2048


def clear_caches() -> None:
    """Drop the per-geometry PSF kernels and NUFFT device tables (device memory:
    ~100 MB of spectra per 2048^2 geometry)."""
    from . import nufft

    _PSF_CACHE.clear()
    nufft._TABLE_CACHE.clear()


def _build(angles: np.ndarray, nd: int, source_side: int, odd_side: int | None = None) -> PsfKernel:
    """The kernel of a geometry; immutable, so kernels of the same geometry (repeated
    reconstructions, the levels of repeated hierarchical solves) are shared."""
    n = int(source_side)
    if n < 1:
        raise ValueError("source side must be positive")
    dev = _lib.device()
    odd = int(odd_side) if odd_side is not None else padded_side_for(n)
    key = (dev.index, n, int(nd), odd, np.asarray(angles, dtype=np.float64).tobytes())
    psf = _PSF_CACHE.get(key)
    if psf is None:
        psf = _PSF_CACHE[key] = _build_new(angles, nd, n, dev, odd)
        while len(_PSF_CACHE) > _PSF_CACHE_SIZE:
            _PSF_CACHE.popitem(last=False)
    else:
        _PSF_CACHE.move_to_end(key)
    return psf


def _build_new(angles: np.ndarray, nd: int, n: int, dev, odd: int) -> PsfKernel:
    lib = _lib.ensure_ready()
    m = fft_side_for(n)
    cs = np.stack([np.cos(angles), np.sin(angles)], axis=1).astype(np.float64)
    d_cs = torch.from_numpy(np.ascontiguousarray(cs)).to(dev)
    h = m // 2 + 1
    pq = torch.empty((h, m, 2), dtype=torch.float32, device=dev)
    bi = torch.empty((h, m), dtype=torch.float32, device=dev)
    ws_bytes = lib.tf_psf_workspace_bytes(m)
    ws = _device.workspace(ws_bytes, tag="psf")
    _lib.check(
        lib.tf_psf_build(n, m, int(angles.size), d_cs.data_ptr(), int(nd), pq.data_ptr(),
                         bi.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_handle()),
        "tf_psf_build",
    )
    ang = np.array(angles, dtype=np.float64)
    ang.setflags(write=False)
    return PsfKernel(padded_side=odd, source_side=n, radial_count=int(nd), pq=pq, bi=bi,
                     has_flip=(nd % 2 == 0), fft_side=m, angles=ang)


def compute_psf(plan_pad, source_side: int) -> PsfKernel:
    """PSF from a plan on a padded grid (toeplitz.py:85-124 contract).

    The plan only supplies the polar sampling; its side must satisfy the
    reference's rules (>= 2N-1 and odd) so callers see the same errors.
    """
    m = plan_pad.grid_side
    if m < 2 * source_side - 1:
        raise ValueError(f"padded side {m} is smaller than 2N-1 = {2 * source_side - 1}")
    if m % 2 == 0:
        raise ValueError("padded grid side must be odd so kernel lags are integers")
    s = plan_pad.sampling
    return _build(np.asarray(s.angles), s.radial_count, source_side, odd_side=m)


def build_psf(sampling: PolarSampling, source_side: int, tolerance: float = 1e-6,
              oversampling: float = 2.0) -> PsfKernel:
    """Kernel for ``sampling`` on an N x N grid (toeplitz.py:127-131)."""
    _check_tolerance(tolerance, oversampling)
    return _build(np.asarray(sampling.angles), sampling.radial_count, source_side)


def apply_stack(psf: PsfKernel, x: torch.Tensor, out: torch.Tensor | None = None,
                aux: torch.Tensor | None = None, alpha: float = 1.0,
                beta: float = 0.0) -> torch.Tensor:
    """out = alpha * K x + beta * aux on a contiguous fp32 device stack (Z, N, N)."""
    lib = _lib.ensure_ready()
    n, m = psf.source_side, psf.fft_side
    if x.dim() != 3 or x.shape[1] != n or x.shape[2] != n:
        raise ValueError(f"image side {x.shape[-1]} does not match kernel source side {n}")
    if not x.is_contiguous() or x.dtype != torch.float32:
        raise ValueError("apply_stack needs a contiguous fp32 tensor")
    z = x.shape[0]
    if out is None:
        out = torch.empty_like(x)
    if aux is not None and (aux.shape != x.shape or not aux.is_contiguous()):
        raise ValueError("aux must match the input stack")
    per_slice = lib.tf_toeplitz_workspace_bytes(n, m, 1)
    chunk = max(1, min(z, _MAX_CHUNK_BYTES // per_slice))
    ws = _device.workspace(per_slice * chunk)
    _lib.check(
        lib.tf_toeplitz_apply(x.data_ptr(), out.data_ptr(), _lib.ptr(aux), float(alpha),
                              float(beta), z, n, m, psf.pq.data_ptr(), psf.bi.data_ptr(),
                              int(psf.has_flip), ws.data_ptr(), per_slice * chunk,
                              _lib.stream_handle()),
        "tf_toeplitz_apply",
    )
    return out


def _check_side(psf: PsfKernel, side: int) -> None:
    if side != psf.source_side:
        raise ValueError(f"image side {side} does not match kernel source side {psf.source_side}")


def toeplitz_apply(psf: PsfKernel, f):
    """R*R f for an ImageGrid, Volume, array or CUDA tensor (toeplitz.py:152-165)."""
    kind = _device.host_kind(f)
    if kind is not None:  # host float64 in and out: chunked, overlapped transfers
        arr = f.data if kind in ("image", "volume") else f
        _check_side(psf, arr.shape[-1])
        if arr.shape[-2] != arr.shape[-1]:
            raise ValueError(f"image side {arr.shape[-1]} does not match kernel source side")
        return _device.pipelined_host_map(arr, kind, lambda z0, z1, x: apply_stack(psf, x))
    x, kind = _device.as_stack(f)
    _check_side(psf, x.shape[-1])
    return _device.wrap_like(kind, apply_stack(psf, x))


class FidelityContext:
    """Per-(geometry, data) precomputation reused across iterations (toeplitz.py:173-197).

    Constructed as the reference does, ``FidelityContext(psf, rstar_g, g_norm_sq)``
    with ``rstar_g`` an ImageGrid / Volume (or float64 array); it is uploaded once
    and kept on the device as the fp32 (Z, N, N) stack ``rstar``.  Internal callers
    pass the device stack directly (``rstar_g`` may be a CUDA tensor, or use the
    ``rstar=`` keyword).  ``rstar_g`` returns the reference's host view (the
    object given, or one materialised on demand).  Immutable.
    """

    __slots__ = ("psf", "rstar", "g_norm_sq", "_host")

    def __init__(self, psf: PsfKernel, rstar_g=None, g_norm_sq: float = 0.0, *, rstar=None):
        if (rstar_g is None) == (rstar is None):
            raise TypeError("FidelityContext needs exactly one of rstar_g / rstar")
        src = rstar_g if rstar_g is not None else rstar
        host = src if isinstance(src, (ImageGrid, Volume)) else None
        if isinstance(src, torch.Tensor) and src.is_cuda:
            dev = src.to(torch.float32)
            dev = (dev[None] if dev.dim() == 2 else dev).contiguous()
        else:
            dev, _ = _device.as_stack(src, "rstar_g")
        if dev.shape[-1] != psf.source_side:
            raise ValueError("adjoint image side does not match PSF source side")
        for name, val in (("psf", psf), ("rstar", dev), ("g_norm_sq", float(g_norm_sq)),
                          ("_host", host)):
            object.__setattr__(self, name, val)

    def __setattr__(self, name, value):
        raise AttributeError("FidelityContext is immutable")

    def __repr__(self):
        return (f"FidelityContext(psf=<N={self.psf.source_side}>, slices={self.slices}, "
                f"g_norm_sq={self.g_norm_sq!r})")

    @property
    def slices(self) -> int:
        return self.rstar.shape[0]

    @property
    def side(self) -> int:
        return self.rstar.shape[-1]

    @property
    def rstar_g(self):
        if self._host is not None:
            return self._host
        host = self.rstar.detach().to("cpu", torch.float64).numpy()
        return ImageGrid(host[0]) if host.shape[0] == 1 else Volume(host)

    def rstar_array(self) -> np.ndarray:
        return self.rstar.detach().to("cpu", torch.float64).numpy()


def fidelity_context(recon_plan, psf: PsfKernel, sino: Sinogram) -> FidelityContext:
    """R*g (GPU NUFFT back-projection) and ||g||^2 (toeplitz.py:200-207)."""
    from .radon import _sampling_matches, back_project_stack

    _sampling_matches(recon_plan, sino.angles, sino.detector_bins)
    if recon_plan.grid_side != psf.source_side:
        raise ValueError("reconstruction plan side does not match PSF source side")
    rstar = back_project_stack(recon_plan, sino.data)
    return FidelityContext(psf, rstar=rstar, g_norm_sq=float(np.sum(sino.data ** 2)))


def _fidelity_stack(ctx: FidelityContext, f):
    x, kind = _device.as_stack(f, "estimate")
    if tuple(x.shape) != (ctx.slices, ctx.side, ctx.side):
        raise ValueError(
            f"estimate shape {tuple(x.shape)} does not match data "
            f"({ctx.slices}, {ctx.side}, {ctx.side})"
        )
    return x, kind


def fidelity_loss(ctx: FidelityContext, f) -> float:
    """0.5 <f, Kf> - <f, R*g> + 0.5 g'g (toeplitz.py:226-230)."""
    from .reduce import dot2

    x, _ = _fidelity_stack(ctx, f)
    kf = apply_stack(ctx.psf, x)
    fkf, frg = dot2(x, kf, ctx.rstar)
    return 0.5 * fkf - frg + 0.5 * ctx.g_norm_sq


def fidelity_grad(ctx: FidelityContext, f):
    """K f - R*g, same kind as the input (toeplitz.py:233-241)."""
    kind = _device.host_kind(f)
    if kind is not None:  # host float64 in and out: chunked, overlapped transfers
        arr = f.data if kind in ("image", "volume") else f
        shape = (1,) + arr.shape if arr.ndim == 2 else arr.shape
        if tuple(shape) != (ctx.slices, ctx.side, ctx.side):
            raise ValueError(f"estimate shape {tuple(shape)} does not match data "
                             f"({ctx.slices}, {ctx.side}, {ctx.side})")
        return _device.pipelined_host_map(
            arr, kind, lambda z0, z1, x: apply_stack(ctx.psf, x, aux=ctx.rstar[z0:z1],
                                                     alpha=1.0, beta=-1.0))
    x, kind = _fidelity_stack(ctx, f)
    grad = apply_stack(ctx.psf, x, aux=ctx.rstar, alpha=1.0, beta=-1.0)
    return _device.wrap_like(kind, grad)
