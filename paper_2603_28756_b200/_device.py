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


_CHUNK_ELEMS = 1 << 23  # 64 MB of float64 per staged copy (32 MB page-locked fp32
# stages: a process's first 2048^3-sinogram upload spent ~0.14 s pinning 2 x 128 MB)
# host float64 inputs are narrowed to fp32 by the staging threads (round to
# nearest, bit-identical to narrowing on the device, half the upload bytes);
# 4.3 GB float64 -> device: 0.09 s with 8 threads, 0.08 s with 16
_STAGE_THREADS = min(16, os.cpu_count() or 1)
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
    # narrowed to fp32 by the host threads while staging (see pipelined_host_map)
    tdt = torch.float32
    stages = [torch.empty(chunk, dtype=tdt, pin_memory=True) for _ in range(2)]
    events = [None, None]
    stream = torch.cuda.current_stream()

    def fill(stage, lo, hi):
        part = (hi - lo) // _STAGE_THREADS + 1
        view = stage.numpy()
        futs = [_pool().submit(np.copyto, view[a - lo:min(hi, a + part) - lo], flat[a:min(hi, a + part)],
                               "same_kind")
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


_OUT_CHUNK = 1 << 23  # 64 MB of float64 per staged chunk


def to_host64(t: torch.Tensor) -> np.ndarray:
    """fp32 device tensor -> float64 host array (widened on the device, chunked).

    The result lives in page-locked memory from torch's caching host allocator
    (the returned array keeps its tensor alive): the device->host copy runs at
    link speed and, once the caller drops a result, the next call of that size
    reuses the block (the first one pays for pinning it).  When page-locked
    memory runs out the copy goes through two small staged chunks into a
    pageable array."""
    src = t.detach().reshape(-1)
    try:
        out = torch.empty(tuple(t.shape), dtype=torch.float64, pin_memory=True)
    except RuntimeError:  # pinned memory exhausted: pageable fallback of the host buffer
        return _to_host64_staged(src).reshape(tuple(t.shape))
    dst = out.reshape(-1)
    for lo in range(0, src.numel(), _CHUNK_ELEMS):
        hi = min(src.numel(), lo + _CHUNK_ELEMS)
        dst[lo:hi].copy_(src[lo:hi].to(torch.float64), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out.numpy()


def _to_host64_staged(src: torch.Tensor) -> np.ndarray:
    out = np.empty(src.numel(), dtype=np.float64)
    stages = [torch.empty(_OUT_CHUNK, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    pending = [None, None]  # (lo, hi, event) of the chunk in each stage

    def drain(b):
        lo, hi, ev = pending[b]
        ev.synchronize()
        view = stages[b].numpy()
        part = (hi - lo) // _STAGE_THREADS + 1
        futs = [_pool().submit(np.copyto, out[a:min(hi, a + part)], view[a - lo:min(hi, a + part) - lo])
                for a in range(lo, hi, part)]
        for f in futs:
            f.result()
        pending[b] = None

    for i, lo in enumerate(range(0, src.numel(), _OUT_CHUNK)):
        hi = min(src.numel(), lo + _OUT_CHUNK)
        b = i % 2
        if pending[b] is not None:
            drain(b)
        stages[b][:hi - lo].copy_(src[lo:hi].to(torch.float64), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        pending[b] = (lo, hi, ev)
    for b in sorted(range(2), key=lambda b: pending[b][0] if pending[b] else 0):
        if pending[b] is not None:
            drain(b)
    return out


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


def host_kind(f) -> str | None:
    """The reference kind of a host input ('image', 'volume', 'array2', 'array3'), or
    None for CUDA tensors / anything to be handled by ``as_stack``."""
    if isinstance(f, ImageGrid):
        return "image"
    if isinstance(f, Volume):
        return "volume"
    if isinstance(f, np.ndarray) and f.ndim in (2, 3):
        return "array2" if f.ndim == 2 else "array3"
    return None


def _wrap_host(kind: str, host: np.ndarray):
    if kind == "image":
        return ImageGrid._owned(host[0])
    if kind == "volume":
        return Volume._owned(host)
    if kind == "array2":
        return host[0]
    return host


_PIPE_SLICE_BYTES = 256 << 20
_streams: dict = {}


def _pipe_streams(dev):
    st = _streams.get(dev.index)
    if st is None:
        st = _streams[dev.index] = tuple(torch.cuda.Stream(device=dev) for _ in range(3))
    return st


def pipelined_host_map(arr: np.ndarray, kind: str, fn):
    """out[z] = fn(z0, z1, x_dev[z0:z1]) for a float64 host stack, chunked over slices
    and pipelined over three streams: the host threads fill a page-locked stage and
    the copy stream uploads chunk i+1 while the compute stream runs ``fn`` on chunk i
    and the download stream returns chunk i-1 into a page-locked float64 result
    (PCIe/NVLink-C2C full duplex).  ``fn`` must return a new (z1-z0, ...) fp32
    device tensor.  Returns the result in the caller's kind."""
    dev = _lib.device()
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    stack = arr[None] if arr.ndim == 2 else arr
    z = stack.shape[0]
    plane = int(np.prod(stack.shape[1:]))
    step = max(1, min(z, _PIPE_SLICE_BYTES // max(1, plane * 8)))
    try:
        out = torch.empty(stack.shape, dtype=torch.float64, pin_memory=True)
    except RuntimeError:
        out = torch.empty(stack.shape, dtype=torch.float64)
    # the host threads narrow to fp32 while staging (round to nearest, as the device
    # conversion would): half the upload bytes and half the staging writes
    sdt = torch.float32
    stages = [torch.empty(step * plane, dtype=sdt, pin_memory=True) for _ in range(2)]
    staged = [None, None]
    caller = torch.cuda.current_stream()
    s_up, s_cmp, s_dn = _pipe_streams(dev)
    for q in (s_up, s_cmp, s_dn):
        q.wait_stream(caller)
    flat = stack.reshape(z, plane)
    for i, z0 in enumerate(range(0, z, step)):
        z1 = min(z, z0 + step)
        b = i % 2
        if staged[b] is not None:
            staged[b].synchronize()  # stage b's previous upload has been read
        view = stages[b].numpy()[: (z1 - z0) * plane]
        src = flat[z0:z1].reshape(-1)
        part = -(-src.size // _STAGE_THREADS)
        futs = [_pool().submit(np.copyto, view[a:a + part], src[a:a + part], "same_kind")
                for a in range(0, src.size, part)]
        for fu in futs:
            fu.result()
        with torch.cuda.stream(s_up):
            xs = stages[b][: view.size].to(dev, non_blocking=True)
            x = xs.reshape((z1 - z0,) + stack.shape[1:]).to(torch.float32)
            ev = torch.cuda.Event()
            ev.record(s_up)
            staged[b] = ev
        s_cmp.wait_stream(s_up)
        x.record_stream(s_cmp)
        with torch.cuda.stream(s_cmp):
            y = fn(z0, z1, x)
        s_dn.wait_stream(s_cmp)
        y.record_stream(s_dn)
        with torch.cuda.stream(s_dn):
            out[z0:z1].copy_(y.to(torch.float64), non_blocking=True)
    caller.wait_stream(s_dn)
    s_dn.synchronize()
    return _wrap_host(kind, out.numpy())
