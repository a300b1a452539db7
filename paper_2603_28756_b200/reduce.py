"""fp64 reductions over device stacks through the C-ABI (deterministic order)."""

from __future__ import annotations

import torch

from . import _device, _lib


def dot2(x: torch.Tensor, a: torch.Tensor, b: torch.Tensor | None = None):
    """(sum x*a, sum x*b) accumulated in fp64 on the device; b may be None."""
    lib = _lib.ensure_ready()
    for t in (x, a) + ((b,) if b is not None else ()):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise ValueError("dot2 needs contiguous fp32 CUDA tensors")
        if t.numel() != x.numel():
            raise ValueError("dot2 operands differ in size")
    out = torch.empty(2, dtype=torch.float64, device=x.device)
    wsb = lib.tf_reduce_workspace_bytes()
    ws = _device.workspace(wsb, tag="reduce")
    _lib.check(lib.tf_dot2(x.data_ptr(), a.data_ptr(), _lib.ptr(b), x.numel(), out.data_ptr(),
                           ws.data_ptr(), _lib.stream_handle()), "tf_dot2")
    vals = out.tolist()
    return vals[0], vals[1]
