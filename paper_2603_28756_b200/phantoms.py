"""Synthetic test objects (input generators for tests and benchmarks).

Numerically identical to the reference phantoms (tomoforge/geometry.py:216-281):
the modified Shepp-Logan ellipse table on normalised pixel centres, with an
ellipsoidal taper along z for volumes, and a centred disk.
"""

from __future__ import annotations

import numpy as np

# value, semi-axes (a, b), centre (x0, y0), rotation (degrees): the standard
# modified (high-contrast) Shepp-Logan table
_TABLE = np.array([
    [1.00, 0.6900, 0.9200, 0.00, 0.0000, 0.0],
    [-0.80, 0.6624, 0.8740, 0.00, -0.0184, 0.0],
    [-0.20, 0.1100, 0.3100, 0.22, 0.0000, -18.0],
    [-0.20, 0.1600, 0.4100, -0.22, 0.0000, 18.0],
    [0.10, 0.2100, 0.2500, 0.00, 0.3500, 0.0],
    [0.10, 0.0460, 0.0460, 0.00, 0.1000, 0.0],
    [0.10, 0.0460, 0.0460, 0.00, -0.1000, 0.0],
    [0.10, 0.0460, 0.0230, -0.08, -0.6050, 0.0],
    [0.10, 0.0230, 0.0230, 0.00, -0.6060, 0.0],
    [0.10, 0.0230, 0.0460, 0.06, -0.6050, 0.0],
])
_Z_EXTENT = 0.95  # half-height of the ellipsoidal taper (normalised)


def _slice(side: int, scale: float) -> np.ndarray:
    """One phantom slice with every ellipse scaled by ``scale`` (0 -> empty)."""
    img = np.zeros((side, side))
    if scale <= 0.0:
        return img
    c = (2.0 * np.arange(side) - (side - 1.0)) / side  # pixel centres in (-1, 1)
    gx, gy = np.meshgrid(c, c, indexing="ij")
    for val, a, b, x0, y0, deg in _TABLE:
        cs, sn = np.cos(np.deg2rad(deg)), np.sin(np.deg2rad(deg))
        u, v = gx - x0 * scale, gy - y0 * scale
        inside = ((u * cs + v * sn) / (a * scale)) ** 2 + ((v * cs - u * sn) / (b * scale)) ** 2
        img[inside <= 1.0] += val
    return np.maximum(img, 0.0)


def shepp_logan(side: int, three_d: bool = False, slices: int = 1):
    """Shepp-Logan head phantom: an ImageGrid, or a Volume tapered along z."""
    from .geometry import ImageGrid, Volume

    if side < 8:
        raise ValueError("phantom side must be at least 8")
    if not three_d:
        return ImageGrid(_slice(side, 1.0))
    if slices < 1:
        raise ValueError("3D phantom needs at least one slice")
    zc = np.zeros(1) if slices == 1 else (2.0 * np.arange(slices) - (slices - 1.0)) / slices
    scales = np.sqrt(np.maximum(0.0, 1.0 - (zc / _Z_EXTENT) ** 2))
    return Volume(np.stack([_slice(side, float(s)) for s in scales]))


def shepp_logan_slab(side: int, slices: int, z_begin: int, z_end: int, device=None):
    """Slices [z_begin, z_end) of ``shepp_logan(side, three_d=True, slices=slices)``
    evaluated on the device in float64 (same pixel centres, table and taper; returns
    an fp32 (z_end - z_begin, side, side) tensor).  Input generator for volumes too
    large for host numpy (C4: 2048^3)."""
    import torch

    dev = torch.device(device) if device is not None else torch.device("cuda")
    zc = np.zeros(1) if slices == 1 else (2.0 * np.arange(slices) - (slices - 1.0)) / slices
    scales = np.sqrt(np.maximum(0.0, 1.0 - (zc / _Z_EXTENT) ** 2))[z_begin:z_end]
    c = torch.from_numpy((2.0 * np.arange(side) - (side - 1.0)) / side).to(dev)
    gx, gy = c[:, None], c[None, :]
    out = torch.zeros((z_end - z_begin, side, side), dtype=torch.float32, device=dev)
    for k, sc in enumerate(scales):
        if sc <= 0.0:
            continue
        img = torch.zeros((side, side), dtype=torch.float64, device=dev)
        for val, a, b, x0, y0, deg in _TABLE:
            cs, sn = np.cos(np.deg2rad(deg)), np.sin(np.deg2rad(deg))
            u, v = gx - x0 * sc, gy - y0 * sc
            inside = ((u * cs + v * sn) / (a * sc)) ** 2 + ((v * cs - u * sn) / (b * sc)) ** 2
            img += torch.where(inside <= 1.0, val, 0.0)
        out[k] = img.clamp_min_(0.0)
    return out


def disk_phantom(side: int, radius: float, value: float = 1.0):
    """``value`` at pixel centres strictly inside ``radius``, zero elsewhere."""
    from .geometry import ImageGrid

    if not 0.0 < radius <= side / 2.0:
        raise ValueError(f"radius must be in (0, side/2], got {radius}")
    r = np.arange(side) - (side - 1) / 2.0
    return ImageGrid(np.where(np.add.outer(r * r, r * r) < radius * radius, float(value), 0.0))
