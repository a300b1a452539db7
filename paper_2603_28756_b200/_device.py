"""Host <-> device conversion and workspace management for the operator API.

Reference-kind inputs (numpy float64 arrays, ImageGrid, Volume) are copied to
fp32 CUDA tensors at the boundary and results come back as float64 numpy of the
same kind (the reference contract, tomoforge/toeplitz.py:152-165); CUDA
tensors pass through without copies and results stay on the device.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .geometry import ImageGrid, Volume

_workspaces: dict = {}


def workspace(nbytes: int, tag: str = "main") -> torch.Tensor:
    """A cached uint8 device buffer of at least ``nbytes`` (grown on demand)."""
    dev = _lib.device()
    key = (dev.index, tag)
    buf = _workspaces.get(key)
    if buf is None or buf.numel() < nbytes:
        _workspaces.pop(key, None)
        buf = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=dev)
        _workspaces[key] = buf
    return buf


def release_workspaces() -> None:
    _workspaces.clear()


def is_device_tensor(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def as_stack(f, what: str = "input"):
    """Return (device fp32 (Z, N, N) contiguous tensor, kind) for any accepted input.

    kind is one of 'image', 'volume', 'array2', 'array3', 'tensor2', 'tensor3'.
    """
    if isinstance(f, ImageGrid):
        return to_device(f.data[None]), "image"
    if isinstance(f, Volume):
        return to_device(f.data), "volume"
    if isinstance(f, torch.Tensor):
        t = f
        if not t.is_cuda:
            t = t.to(_lib.device())
        t = t.to(torch.float32).contiguous()
        if t.dim() == 2:
            return t[None], "tensor2"
        if t.dim() == 3:
            return t, "tensor3"
        raise ValueError(f"{what} must be 2D or 3D, got shape {tuple(t.shape)}")
    arr = np.asarray(f, dtype=np.float64)
    if arr.ndim == 2:
        return to_device(arr[None]), "array2"
    if arr.ndim == 3:
        return to_device(arr), "array3"
    raise ValueError(f"{what} must be 2D or 3D, got shape {arr.shape}")


_CHUNK_ELEMS = 1 << 25  # 256 MB of float64 per staged copy


def to_device(arr: np.ndarray) -> torch.Tensor:
    """float64 (or any real) host array -> contiguous fp32 device tensor.

    The host array is copied as is (no host-side conversion pass) in chunks of
    256 MB and narrowed to fp32 on the device."""
    arr = np.ascontiguousarray(arr)
    dev = _lib.device()
    if arr.dtype == np.float32:
        return torch.from_numpy(arr).to(dev)
    if arr.dtype != np.float64:
        arr = arr.astype(np.float64)
    out = torch.empty(arr.shape, dtype=torch.float32, device=dev)
    src = torch.from_numpy(arr).reshape(-1)
    dst = out.reshape(-1)
    for lo in range(0, src.numel(), _CHUNK_ELEMS):
        hi = min(src.numel(), lo + _CHUNK_ELEMS)
        dst[lo:hi].copy_(src[lo:hi].to(dev))
    return out


def to_host64(t: torch.Tensor) -> np.ndarray:
    """fp32 device tensor -> float64 host array (widened on the device, chunked).

    The result lives in page-locked memory from torch's caching host allocator
    (the returned array keeps its tensor alive), so the device->host copy runs
    at full link speed and repeated calls reuse the pinned block."""
    try:
        out = torch.empty(tuple(t.shape), dtype=torch.float64, pin_memory=True)
    except RuntimeError:  # pinned memory exhausted: pageable fallback of the host buffer
        out = torch.empty(tuple(t.shape), dtype=torch.float64)
    dst = out.reshape(-1)
    src = t.detach().reshape(-1)
    for lo in range(0, src.numel(), _CHUNK_ELEMS):
        hi = min(src.numel(), lo + _CHUNK_ELEMS)
        dst[lo:hi].copy_(src[lo:hi].to(torch.float64), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out.numpy()


def wrap_like(kind: str, t: torch.Tensor):
    """Return the device stack ``t`` in the caller's kind."""
    if kind == "tensor3":
        return t
    if kind == "tensor2":
        return t[0]
    host = to_host64(t)
    if kind == "image":
        return ImageGrid._owned(host[0])
    if kind == "volume":
        return Volume._owned(host)
    if kind == "array2":
        return host[0]
    return host
