"""Host <-> device conversion and workspace management for the operator API.

Reference-kind inputs (numpy float64 arrays, ImageGrid, Volume) are copied to
fp32 CUDA tensors at the boundary and results come back as float64 numpy of the
same kind (the reference contract, tomoforge/toeplitz.py:152-165); CUDA
tensors pass through without copies and results stay on the device.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

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


_STAGE_THREADS = min(8, os.cpu_count() or 1)
_stage_pool = None


def _pool():
    global _stage_pool
    if _stage_pool is None:
        _stage_pool = ThreadPoolExecutor(max_workers=_STAGE_THREADS)
    return _stage_pool


def to_device(arr: np.ndarray) -> torch.Tensor:
    """float64 (or any real) host array -> contiguous fp32 device tensor.

    Large arrays go through two page-locked staging buffers (torch's caching host
    allocator): host threads fill chunk i+1 (numpy copies release the GIL) while
    chunk i is in flight to the device, where it is narrowed to fp32."""
    arr = np.ascontiguousarray(arr)
    dev = _lib.device()
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    out = torch.empty(arr.shape, dtype=torch.float32, device=dev)
    flat = arr.reshape(-1)
    dst = out.reshape(-1)
    total = flat.size
    if total * flat.itemsize < (64 << 20):  # small: one plain copy
        if not flat.flags.writeable:
            flat = flat.copy()
        dst.copy_(torch.from_numpy(flat).to(dev))
        return out
    chunk = _CHUNK_ELEMS
    tdt = torch.float64 if flat.dtype == np.float64 else torch.float32
    stages = [torch.empty(chunk, dtype=tdt, pin_memory=True) for _ in range(2)]
    events = [None, None]
    stream = torch.cuda.current_stream()

    def fill(stage, lo, hi):
        part = (hi - lo) // _STAGE_THREADS + 1
        view = stage.numpy()
        futs = [_pool().submit(np.copyto, view[a - lo:min(hi, a + part) - lo], flat[a:min(hi, a + part)])
                for a in range(lo, hi, part)]
        for f in futs:
            f.result()

    for i, lo in enumerate(range(0, total, chunk)):
        hi = min(total, lo + chunk)
        b = i % 2
        if events[b] is not None:
            events[b].synchronize()  # the stage's previous upload has finished reading it
        fill(stages[b], lo, hi)
        dev_chunk = stages[b][:hi - lo].to(dev, non_blocking=True)
        dst[lo:hi].copy_(dev_chunk)
        events[b] = torch.cuda.Event()
        events[b].record(stream)
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
