"""The C-ABI library loads and exports every entry point include/*.h declares (CPU only:
no compute calls)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    names = []
    for h in sorted((ROOT / "include").glob("*.h")):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names += re.findall(r"\b(tf_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_28756_b200.build import build_library

    return ctypes.CDLL(str(build_library()))


def test_header_declares_entry_points():
    assert len(_declared()) >= 15


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, f"not exported: {missing}"


def test_bindings_match_header():
    from paper_2603_28756_b200 import _lib

    assert sorted(_lib.declared_symbols()) == _declared()


def test_host_only_entry_points(lib):
    lib.tf_fft_side.restype = ctypes.c_int
    assert lib.tf_fft_side(2048) == 4096
    assert lib.tf_fft_side(256) == 512
    # 5 * 2^k sides where smaller (radix-5 step): the C5 levels 640 / 1280 / 2560
    assert [lib.tf_fft_side(n) for n in (640, 1280, 2560, 600, 300)] == [1280, 2560, 5120, 1280, 1024]
    assert lib.tf_fft_side(0) == -1
    lib.tf_last_error.restype = ctypes.c_char_p
    assert b"positive" in lib.tf_last_error()
    lib.tf_toeplitz_workspace_bytes.restype = ctypes.c_longlong
    lib.tf_toeplitz_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_longlong]
    assert lib.tf_toeplitz_workspace_bytes(2048, 4096, 1) == 2049 * 4 * 512 * 8
