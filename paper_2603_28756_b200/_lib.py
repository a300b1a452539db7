"""ctypes binding of the in-tree C-ABI library ``libtomoforge_b200.so``.

The declarations mirror ``include/tomoforge_b200.h``.  Every entry point
returns 0 on success, -1 (bad argument -> ``ValueError``), -2 (CUDA error ->
``RuntimeError``) or -3 (unsupported -> ``NotImplementedError``).  There is no
CPU fallback: importing a compute wrapper without the built library or without
a CUDA device raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("TF_LIB_PATH", _HERE / "libtomoforge_b200.so"))

_c_void_p = ctypes.c_void_p
_c_int = ctypes.c_int
_c_ll = ctypes.c_longlong
_c_float = ctypes.c_float
_c_double = ctypes.c_double

# name -> (restype, argtypes); must match include/tomoforge_b200.h
_SIGNATURES = {
    "tf_last_error": (ctypes.c_char_p, []),
    "tf_version": (_c_int, []),
    "tf_init": (_c_int, []),
    "tf_fft_side": (_c_int, [_c_int]),
    "tf_toeplitz_workspace_bytes": (_c_ll, [_c_int, _c_int, _c_ll]),
    "tf_psf_workspace_bytes": (_c_ll, [_c_int]),
    "tf_psf_build": (_c_int, [_c_int, _c_int, _c_int, _c_void_p, _c_int, _c_void_p, _c_void_p,
                              _c_void_p, _c_ll, _c_void_p]),
    "tf_psf_kernel": (_c_int, [_c_int, _c_int, _c_void_p, _c_int, _c_void_p, _c_void_p]),
    "tf_toeplitz_apply": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_float, _c_float, _c_ll,
                                   _c_int, _c_int, _c_void_p, _c_void_p, _c_int, _c_void_p,
                                   _c_ll, _c_void_p]),
    "tf_reduce_workspace_bytes": (_c_ll, []),
    "tf_dot2": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_ll, _c_void_p, _c_void_p,
                         _c_void_p]),
    "tf_prior_workspace_bytes": (_c_ll, [_c_int, _c_int]),
    "tf_prior_update": (_c_int, [_c_void_p] * 10 + [_c_int, _c_int, _c_int, _c_float, _c_float, _c_float,
                                                    _c_int, _c_int, _c_int, _c_double, _c_double,
                                                    _c_double, _c_double, _c_void_p, _c_void_p,
                                                    _c_void_p, _c_void_p]),
    "tf_prior_update_dc": (_c_int, [_c_void_p] * 10 + [_c_int, _c_int, _c_int, _c_float, _c_void_p,
                                                       _c_float, _c_float, _c_int, _c_int, _c_int,
                                                       _c_double, _c_double, _c_double, _c_double,
                                                       _c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "tf_prior_update_if": (_c_int, [_c_void_p] * 10 + [_c_int, _c_int, _c_int, _c_void_p, _c_float,
                                                       _c_float, _c_int, _c_double, _c_double,
                                                       _c_double, _c_double, _c_void_p, _c_void_p,
                                                       _c_void_p, _c_void_p, _c_void_p]),
    "tf_prior_energy_update": (_c_int, [_c_void_p] * 10 + [_c_int, _c_int, _c_int, _c_void_p,
                                                           _c_float, _c_float, _c_int, _c_int,
                                                           _c_double, _c_double, _c_double,
                                                           _c_double] + [_c_void_p] * 7),
    "tf_upsample3": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_int, _c_int, _c_int,
                              _c_int, _c_void_p, _c_void_p, _c_int, _c_void_p, _c_void_p, _c_int,
                              _c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_void_p]),
    "tf_solver_decide": (_c_int, [_c_void_p] * 4 + [_c_double, _c_int, _c_int, _c_double,
                                                    _c_void_p]),
    "tf_energy_fid": (_c_int, [_c_void_p] * 6 + [_c_int, _c_int, _c_int, _c_int, _c_int, _c_double,
                                                 _c_double, _c_double, _c_double, _c_void_p,
                                                 _c_void_p, _c_void_p, _c_void_p]),
    "tf_detector_rows": (_c_int, [_c_void_p, _c_ll, _c_int, _c_int, _c_void_p, _c_int, _c_int,
                                  _c_float, _c_void_p, _c_void_p]),
    "tf_nufft_workspace_bytes": (_c_ll, [_c_int, _c_ll]),
    "tf_nufft_type1": (_c_int, [_c_void_p, _c_ll, _c_ll, _c_int, _c_int, _c_int] + [_c_void_p] * 7
                       + [_c_float, _c_int, _c_void_p, _c_void_p, _c_ll, _c_void_p]),
    "tf_halo_signal": (_c_int, [_c_void_p, ctypes.c_ulonglong, _c_void_p]),
    "tf_halo_wait": (_c_int, [_c_void_p, _c_void_p, ctypes.c_ulonglong, _c_void_p]),
    "tf_nufft_plan_weights": (_c_int, [_c_void_p, _c_ll, _c_int, _c_int, _c_double, _c_void_p,
                                       _c_void_p, _c_void_p]),
    "tf_nufft_type2_workspace_bytes": (_c_ll, [_c_int, _c_int, _c_ll]),
    "tf_nufft_type2": (_c_int, [_c_void_p, _c_ll, _c_int, _c_int, _c_int] + [_c_void_p] * 5
                       + [_c_ll, _c_void_p, _c_void_p, _c_ll, _c_void_p]),
    "tf_detector_rows_inv": (_c_int, [_c_void_p, _c_ll, _c_int, _c_float, _c_void_p, _c_void_p]),
    "tf_direct_dft": (_c_int, [_c_void_p, _c_int, _c_void_p, _c_ll, _c_void_p, _c_void_p]),
    "tf_resample_axis": (_c_int, [_c_void_p, _c_void_p, _c_ll, _c_int, _c_int, _c_ll, _c_void_p,
                                  _c_void_p, _c_int, _c_void_p]),
    "tf_timing_enable": (_c_int, [_c_int]),
    "tf_timing_collect": (_c_int, [_c_void_p, _c_void_p, _c_int]),
}

# kernel timing slots (tf_timing_collect)
TIMER_SLOTS = {"k_rows_fwd": 0, "k_cols_conv": 1, "k_rows_inv": 2}

_lib = None


def load(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and return the C-ABI library; raises if it was not built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the reconstruction kernels)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def declared_symbols():
    return list(_SIGNATURES)


def last_error() -> str:
    msg = load().tf_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = f"{what}: {last_error()}"
    if rc == -1:
        raise ValueError(msg)
    if rc == -3:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


_initialised = set()


def device() -> torch.device:
    """The CUDA device every kernel runs on (the current one)."""
    if not torch.cuda.is_available():
        raise RuntimeError("tomoforge-b200 needs a CUDA device; there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def ensure_ready() -> ctypes.CDLL:
    lib = load()
    dev = device()
    if dev.index not in _initialised:
        check(lib.tf_init(), "tf_init")
        _initialised.add(dev.index)
    return lib


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def timing_enable(on: bool) -> None:
    check(load().tf_timing_enable(1 if on else 0), "tf_timing_enable")


def timing_collect(nslots: int = 16):
    """{slot: (total_ms, launches)} for the events recorded since timing_enable(True)."""
    ms = (ctypes.c_double * nslots)()
    n = (ctypes.c_longlong * nslots)()
    check(load().tf_timing_collect(ctypes.addressof(ms), ctypes.addressof(n), nslots),
          "tf_timing_collect")
    return {i: (ms[i], n[i]) for i in range(nslots) if n[i] > 0}
