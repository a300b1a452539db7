"""Edge-preserving qGGMRF prior over 8/26-neighbour cliques on the GPU.

Drop-in for tomoforge/qggmrf.py.  Same parameter object, stencils, potential
definitions and boundary conventions: cliques leaving the volume are dropped,
halo planes (slab boundaries) are real data for the gradient, and the energy
counts each unordered pair once with pairs into ``halo_hi`` owned by the lower
slab (qggmrf.py:1-19, :142-217).  The gradient and the energy run in the CUDA
kernels of csrc/qggmrf.cu (K4 / K5); the per-element potentials evaluate on the
device with torch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .geometry import ImageGrid, Volume

__all__ = [
    "QggmrfParams",
    "NeighborStencil",
    "stencil_2d",
    "stencil_3d",
    "stencil_for",
    "potential",
    "potential_deriv",
    "prior_grad",
    "prior_energy",
]


@dataclass(frozen=True)
class QggmrfParams:
    """Shape (p, q, T), scale sigma and weight lam (qggmrf.py:43-61)."""

    sigma: float
    lam: float = 0.0
    p: float = 2.0
    q: float = 1.2
    T: float = 1.0

    def __post_init__(self):
        if not (1.0 <= self.q < self.p <= 2.0):
            raise ValueError(f"require 1 <= q < p <= 2, got p={self.p}, q={self.q}")
        if self.T <= 0:
            raise ValueError("transition threshold T must be positive")
        if self.sigma <= 0:
            raise ValueError("sigma must be positive")
        if self.lam < 0:
            raise ValueError("regularization weight must be nonnegative")


@dataclass(frozen=True)
class NeighborStencil:
    """Clique offsets (dz, dy, dx) and inverse-distance weights summing to 1."""

    offsets: tuple
    weights: np.ndarray = field(repr=False)

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=np.float64)
        object.__setattr__(self, "weights", w)
        if len(self.offsets) not in (8, 26):
            raise ValueError("stencil must have 8 (2D) or 26 (3D) offsets")
        if np.any(w <= 0) or abs(w.sum() - 1.0) > 1e-12:
            raise ValueError("weights must be positive and sum to 1")

    def half(self):
        """Lexicographically positive offsets: every unordered pair once."""
        return [(o, w) for o, w in zip(self.offsets, self.weights) if o > (0, 0, 0)]

    @property
    def three_d(self) -> bool:
        return len(self.offsets) == 26

    def class_weights(self) -> np.ndarray:
        """Weights by the number of nonzero offset components (1, 2, 3) -- the
        form the kernels take; rejects stencils that are not distance-isotropic."""
        out = np.zeros(3)
        seen = [None, None, None]
        for o, w in zip(self.offsets, self.weights):
            k = sum(1 for v in o if v != 0) - 1
            if seen[k] is not None and abs(seen[k] - w) > 1e-15 * max(1.0, w):
                raise NotImplementedError("kernels support the inverse-distance 8/26 stencils only")
            seen[k] = w
            out[k] = w
        return out


def _build(three_d: bool) -> NeighborStencil:
    zs = (-1, 0, 1) if three_d else (0,)
    offs = [(a, b, c) for a in zs for b in (-1, 0, 1) for c in (-1, 0, 1) if (a, b, c) != (0, 0, 0)]
    inv = np.array([1.0 / math.sqrt(a * a + b * b + c * c) for a, b, c in offs])
    return NeighborStencil(offsets=tuple(offs), weights=inv / inv.sum())


_S2, _S3 = _build(False), _build(True)


def stencil_2d() -> NeighborStencil:
    return _S2


def stencil_3d() -> NeighborStencil:
    return _S3


def stencil_for(arr) -> NeighborStencil:
    """8-neighbour for single-slice problems, 26 otherwise (qggmrf.py:112-114)."""
    return _S3 if arr.shape[0] > 1 else _S2


def _elementwise(delta, fn):
    if isinstance(delta, torch.Tensor):
        return fn(delta.to(_lib.device(), torch.float64))
    d = torch.as_tensor(np.asarray(delta, dtype=np.float64), device=_lib.device())
    out = fn(d).cpu().numpy()
    return out if out.ndim else float(out)


def potential(params: QggmrfParams, delta):
    """rho(delta) = |d|^p / (p sigma^p) / (1 + (|d|/(T sigma))^(p-q)) (qggmrf.py:117-121)."""
    def fn(d):
        a = d.abs()
        v = (a / (params.T * params.sigma)) ** (params.p - params.q)
        return a ** params.p / (params.p * params.sigma ** params.p) / (1.0 + v)
    return _elementwise(delta, fn)


def potential_deriv(params: QggmrfParams, delta):
    """d rho / d delta (qggmrf.py:124-130)."""
    def fn(d):
        a = d.abs()
        v = (a / (params.T * params.sigma)) ** (params.p - params.q)
        shape = (1.0 + (params.q / params.p) * v) / (1.0 + v) ** 2
        return torch.sign(d) * a ** (params.p - 1.0) / params.sigma ** params.p * shape
    return _elementwise(delta, fn)


def _halo(plane, shape, what):
    if plane is None:
        return None
    if isinstance(plane, torch.Tensor):
        t = plane.to(_lib.device(), torch.float32).contiguous()
    else:
        t = _device.to_device(np.asarray(plane, dtype=np.float64))
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{what} plane shape {tuple(t.shape)} does not match slice shape {tuple(shape)}")
    return t


def _consts(params: QggmrfParams):
    return (float(params.sigma), float(params.p), float(params.q), float(params.T))


def _weights_ptr(stencil: NeighborStencil):
    w = np.ascontiguousarray(stencil.class_weights(), dtype=np.float64)
    return w, w.ctypes.data


def prior_update(params, stencil, f, fp, out, *, kf=None, kfp=None, rstar=None, c=0.0, lam=1.0,
                 inv_L=0.0, nonneg=False, write_grad=False, f_lo=None, f_hi=None, fp_lo=None,
                 fp_hi=None, c_dev=None, gsq_out=None) -> torch.Tensor:
    """K4 launch on device stacks; returns a device fp64 tensor [sum(grad^2)] (or
    writes it to the fp64 device scalar ``gsq_out``).  ``c_dev`` (fp32 device
    scalar) overrides ``c`` on the device (solver_decide)."""
    lib = _lib.ensure_ready()
    z, h, w_ = f.shape
    wsb = lib.tf_prior_workspace_bytes(h, w_)
    ws = _device.workspace(wsb, tag="prior")
    gsq = torch.empty(1, dtype=torch.float64, device=f.device) if gsq_out is None else gsq_out
    w, wp = _weights_ptr(stencil)
    P = _lib.ptr
    _lib.check(lib.tf_prior_update_dc(
        P(f), P(f_lo), P(f_hi), P(fp), P(fp_lo), P(fp_hi), P(kf), P(kfp), P(rstar), P(out), z, h, w_,
        float(c), P(c_dev), float(lam), float(inv_L), int(bool(nonneg)), int(bool(write_grad)),
        int(stencil.three_d), *_consts(params), wp, ws.data_ptr(), gsq.data_ptr(),
        _lib.stream_handle()), "tf_prior_update_dc")
    return gsq


def prior_update_if(params, stencil, f, out, *, kf, rstar, c_dev, only_if, gsq_out, lam, inv_L,
                    nonneg=False, f_lo=None, f_hi=None):
    """K4 at y = f (c = *c_dev, 0 after a restart) run only when *only_if != 0: the
    re-run of the update after a restart decision (tf_prior_update_if).  Writes
    sum grad^2 to the fp64 device scalar ``gsq_out`` (a tensor view)."""
    lib = _lib.ensure_ready()
    z, h, w_ = f.shape
    ws = _device.workspace(lib.tf_prior_workspace_bytes(h, w_), tag="prior")
    w, wp = _weights_ptr(stencil)
    P = _lib.ptr
    _lib.check(lib.tf_prior_update_if(
        P(f), P(f_lo), P(f_hi), P(f), P(f_lo), P(f_hi), P(kf), P(kf), P(rstar), P(out), z, h, w_,
        P(c_dev), float(lam), float(inv_L), int(bool(nonneg)), *_consts(params), wp,
        ws.data_ptr(), gsq_out.data_ptr(), only_if.data_ptr(), _lib.stream_handle()),
        "tf_prior_update_if")


def prior_energy_update(params, stencil, f, fp, out, *, kf, kfp, rstar, state, lam, inv_L,
                        nonneg=False, with_prior=True, f_lo=None, f_hi=None, fp_lo=None,
                        fp_hi=None, energy=None, fid=None, dfid=None, gsq=None):
    """K45 (tf_prior_energy_update): K5's sums for f and the no-restart update of
    the next iterate in one pass; the sums land in the given fp64 device scalars
    (tensor views, or None)."""
    lib = _lib.ensure_ready()
    z, h, w_ = f.shape
    ws = _device.workspace(lib.tf_prior_workspace_bytes(h, w_), tag="prior")
    w, wp = _weights_ptr(stencil)
    P = _lib.ptr
    _lib.check(lib.tf_prior_energy_update(
        P(f), P(f_lo), P(f_hi), P(fp), P(fp_lo), P(fp_hi), P(kf), P(kfp), P(rstar), P(out), z, h,
        w_, P(state), float(lam), float(inv_L), int(bool(nonneg)), int(bool(with_prior)),
        *_consts(params), wp, ws.data_ptr(), P(energy), P(fid), P(dfid), P(gsq),
        _lib.stream_handle()), "tf_prior_energy_update")


def solver_decide(vals, state, c_dev, rec, *, lam, with_prior, restart, tol):
    """Restart / momentum / stop decision of one iteration on the device
    (tf_solver_decide): vals = [E_new, sum grad^2, dfid]; state = [obj, fid,
    prior, t, c] updated in place; c_dev <- next c; rec <- the iteration's record."""
    lib = _lib.ensure_ready()
    P = _lib.ptr
    _lib.check(lib.tf_solver_decide(P(vals), P(state), P(c_dev), P(rec), float(lam),
                                    int(bool(with_prior)), int(bool(restart)), float(tol),
                                    _lib.stream_handle()), "tf_solver_decide")


def energy_fid(params, stencil, fn, *, fn_hi=None, f=None, kfn=None, kf=None, rstar=None,
               with_prior=True):
    """K5 launch; returns a device fp64 tensor [E, <fn, Kfn/2 - R*g>, increment]."""
    lib = _lib.ensure_ready()
    z, h, w_ = fn.shape
    wsb = lib.tf_prior_workspace_bytes(h, w_)
    ws = _device.workspace(wsb, tag="energy")
    out = torch.empty(3, dtype=torch.float64, device=fn.device)
    w, wp = _weights_ptr(stencil)
    P = _lib.ptr
    _lib.check(lib.tf_energy_fid(
        P(fn), P(fn_hi), P(f), P(kfn), P(kf), P(rstar), z, h, w_, int(bool(with_prior)),
        int(stencil.three_d), *_consts(params), wp, ws.data_ptr(), out.data_ptr(),
        _lib.stream_handle()), "tf_energy_fid")
    return out


def prior_grad(params: QggmrfParams, stencil: NeighborStencil, vol, halo_lo=None, halo_hi=None):
    """sum_s b_s rho'(f_v - f_{v+s}) per voxel; same kind as the input (qggmrf.py:172-189)."""
    x, kind = _device.as_stack(vol, "volume")
    shape = x.shape[1:]
    lo = _halo(halo_lo, shape, "halo")
    hi = _halo(halo_hi, shape, "halo")
    out = torch.empty_like(x)
    prior_update(params, stencil, x, x, out, lam=1.0, write_grad=True, f_lo=lo, fp_lo=lo,
                 f_hi=hi, fp_hi=hi)
    return _device.wrap_like(kind, out)


def prior_energy(params: QggmrfParams, stencil: NeighborStencil, vol, halo_hi=None) -> float:
    """Clique energy, each unordered pair once, + pairs into halo_hi (qggmrf.py:192-217)."""
    x, _ = _device.as_stack(vol, "volume")
    hi = _halo(halo_hi, x.shape[1:], "halo")
    return float(energy_fid(params, stencil, x, fn_hi=hi)[0].item())
