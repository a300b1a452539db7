"""Back-projection, ramp filtering and FBP on B200 (adjoint Fourier-slice projector).

Drop-in for the reconstruction-side half of tomoforge/radon.py:
``back_project`` (radon.py:112-121), ``back_project_volume`` (:131-134),
``ramp_filter`` / ``RampFilter`` (:37-52), ``ramp_filter_apply`` (:137-142) and
``fbp`` (:145-160).  The forward projector (``forward_project`` / ``project_volume``,
radon.py:85-100) is the type-2 NUFFT followed by an
inverse detector DFT (k_detector_rows_inv).

Every (slice, angle) row goes through K8 (csrc/nufft.cu, k_detector_rows): a
shared-memory DFT of length Nd, the fftshift, the detector-centring phase, 1/Nd,
the plan's half-pixel phase and -- for FBP -- the |w| ramp and the 1/(2P) scale,
folded into one complex factor per sample.  The samples then go through the
type-1 NUFFT (K7 + grid FFT).  FBP therefore never materialises the filtered
sinogram: filtering the rows with |w| and transforming them again
(radon.py:150-157) is the same as weighting the spectrum once, because the ramp
response is even (its product with a Hermitian row spectrum stays Hermitian).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .geometry import ImageGrid, Sinogram, Volume, radial_frequencies
from .nufft import NufftPlan, type1_stack, type2_stack

__all__ = [
    "RampFilter",
    "ramp_filter",
    "ramp_filter_apply",
    "back_project",
    "back_project_volume",
    "back_project_stack",
    "fbp",
    "fbp_stack",
    "forward_project",
    "forward_project_stack",
    "project_volume",
]

_ROW_CHUNK_BYTES = 1 << 30


@dataclass(frozen=True)
class RampFilter:
    """|w| response on the signed frequency range (radon.py:37-47)."""

    length: int
    response: np.ndarray = field(repr=False)

    def __post_init__(self):
        object.__setattr__(self, "response", np.asarray(self.response, dtype=np.float64))
        if self.response.shape != (self.length,):
            raise ValueError("response length mismatch")


def ramp_filter(length: int) -> RampFilter:
    """radon.py:50-52"""
    return RampFilter(length=length, response=np.abs(radial_frequencies(length)))


def _sampling_matches(p: NufftPlan, angles: np.ndarray, nd: int) -> None:
    """radon.py:75-82"""
    s = p.sampling
    if nd != s.radial_count:
        raise ValueError(f"detector bins {nd} do not match plan radial count {s.radial_count}")
    angles = np.asarray(angles)
    if angles.size != s.angles.size or not np.allclose(angles, s.angles):
        raise ValueError("sinogram angles do not match plan angles")


def _rows_device(data) -> torch.Tensor:
    if isinstance(data, torch.Tensor):
        t = data.to(_lib.device(), torch.float32).contiguous()
    else:
        t = _device.to_device(np.asarray(data, dtype=np.float64))
    if t.dim() == 2:
        t = t[None]
    if t.dim() != 3:
        raise ValueError(f"sinogram rows must be (slices, angles, bins), got {tuple(t.shape)}")
    return t


def _project_samples(p: NufftPlan, rows: torch.Tensor, ramp: bool, scale: float) -> torch.Tensor:
    """K8 mode 0: (Z, P, Nd) rows -> (Z, P*Nd) complex64 samples for type1."""
    lib = _lib.ensure_ready()
    z, n_ang, nd = rows.shape
    out = torch.empty((z, n_ang * nd), dtype=torch.complex64, device=rows.device)
    sph = p.detector_sample_phase()
    _lib.check(lib.tf_detector_rows(rows.data_ptr(), z * n_ang, nd, n_ang, sph.data_ptr(), 0,
                                    int(ramp), float(scale), out.data_ptr(), _lib.stream_handle()),
               "tf_detector_rows")
    return out


def _back_project_device(p: NufftPlan, data, ramp: bool, scale: float) -> torch.Tensor:
    rows = _rows_device(data)
    z, n_ang, nd = rows.shape
    if n_ang != p.sampling.angles.size or nd != p.sampling.radial_count:
        raise ValueError(f"sinogram rows {tuple(rows.shape[1:])} do not match the plan sampling "
                         f"({p.sampling.angles.size}, {p.sampling.radial_count})")
    n = p.grid_side
    out = torch.empty((z, n, n), dtype=torch.float32, device=rows.device)
    per_slice = n_ang * nd * 8
    chunk = max(1, min(z, _ROW_CHUNK_BYTES // max(per_slice, 1)))
    for z0 in range(0, z, chunk):
        z1 = min(z, z0 + chunk)
        samples = _project_samples(p, rows[z0:z1], ramp, scale)
        type1_stack(p, samples, out=out[z0:z1])
    return out


def back_project_stack(p: NufftPlan, data) -> torch.Tensor:
    """R* of every slice of (Z, P, Nd) rows -> (Z, N, N) fp32 device tensor
    (radon.py:124-128 per slice; toeplitz.py:205 uses it for R*g)."""
    return _back_project_device(p, data, ramp=False, scale=1.0)


def fbp_stack(p: NufftPlan, data) -> torch.Tensor:
    """Ramp-filtered back-projection x 1/(2P) -> (Z, N, N) fp32 device tensor."""
    rows = _rows_device(data)
    return _back_project_device(p, rows, ramp=True, scale=1.0 / (2.0 * rows.shape[1]))


def back_project(p: NufftPlan, sino) -> ImageGrid:
    """Adjoint of forward_project for a single-slice sinogram (radon.py:112-121)."""
    n_angles = p.sampling.angles.size
    nd = p.sampling.radial_count
    if isinstance(sino, Sinogram):
        _sampling_matches(p, sino.angles, sino.detector_bins)
        rows = sino.data
    else:
        rows = np.asarray(sino, dtype=np.float64)
        if rows.ndim == 2:
            rows = rows[None]
    if rows.shape != (1, n_angles, nd):
        raise ValueError(f"expected single-slice sinogram of shape (1, {n_angles}, {nd})")
    img = back_project_stack(p, rows)
    return ImageGrid._owned(_device.to_host64(img[0]))


def back_project_volume(p: NufftPlan, sino: Sinogram) -> Volume:
    """Adjoint projection of every slice of a stacked sinogram (radon.py:131-134)."""
    _sampling_matches(p, sino.angles, sino.detector_bins)
    return Volume._owned(_device.to_host64(back_project_stack(p, sino.data)))


def ramp_filter_apply(sino: Sinogram) -> Sinogram:
    """Circular |w| filtering of every (slice, angle) row (radon.py:137-142; K8 mode 1)."""
    lib = _lib.ensure_ready()
    rows = _rows_device(sino.data)
    z, n_ang, nd = rows.shape
    out = torch.empty_like(rows)
    _lib.check(lib.tf_detector_rows(rows.data_ptr(), z * n_ang, nd, n_ang, None, 1, 1, 1.0,
                                    out.data_ptr(), _lib.stream_handle()), "tf_detector_rows")
    return Sinogram(angles=sino.angles, data=out.to("cpu", torch.float64).numpy())


def fbp(p: NufftPlan, sino: Sinogram):
    """Filtered back-projection with the 1/(2P) scale (radon.py:145-160): an
    ImageGrid for a single slice, a Volume otherwise."""
    _sampling_matches(p, sino.angles, sino.detector_bins)
    vol = _device.to_host64(fbp_stack(p, sino.data))
    return ImageGrid._owned(vol[0]) if vol.shape[0] == 1 else Volume._owned(vol)


def forward_project_stack(p: NufftPlan, images) -> torch.Tensor:
    """(Z, N, N) images -> (Z, P, Nd) fp32 device projection rows (radon.py:85-96 per slice)."""
    lib = _lib.ensure_ready()
    x = images if isinstance(images, torch.Tensor) else _device.to_device(
        np.asarray(images, dtype=np.float64))
    if x.dim() == 2:
        x = x[None]
    samples = type2_stack(p, x.to(_lib.device()), factor="project")
    n_ang, nd = p.sampling.angles.size, p.sampling.radial_count
    rows = torch.empty((x.shape[0], n_ang, nd), dtype=torch.float32, device=samples.device)
    _lib.check(lib.tf_detector_rows_inv(samples.data_ptr(), x.shape[0] * n_ang, nd, 1.0,
                                        rows.data_ptr(), _lib.stream_handle()),
               "tf_detector_rows_inv")
    return rows


def forward_project(p: NufftPlan, image) -> Sinogram:
    """Parallel-beam projection of one slice (radon.py:85-96)."""
    arr = image.data if isinstance(image, ImageGrid) else np.asarray(image, dtype=np.float64)
    rows = forward_project_stack(p, arr[None])
    return Sinogram(angles=p.sampling.angles, data=_device.to_host64(rows))


def project_volume(p: NufftPlan, vol: Volume) -> Sinogram:
    """Slice-by-slice forward projection of a volume (radon.py:99-103)."""
    return Sinogram(angles=p.sampling.angles, data=_device.to_host64(forward_project_stack(p, vol.data)))
