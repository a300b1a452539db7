"""Build the in-tree C-ABI library with nvcc for sm_100a (no JIT, no torch extension).

Each ``csrc/*.cu`` is its own translation unit, compiled in parallel
(``-gencode arch=compute_100a,code=sm_100a -lineinfo``) and linked into
``libtomoforge_b200.so``.  Objects go to ``build/`` (git-ignored).
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
# tuning builds: TF_BUILD_DEFINES="-DTF_TW_MODE=2" TF_BUILD_OUT=/path/lib.so (separate objects)
_DEFINES = os.environ.get("TF_BUILD_DEFINES", "").split()
LIB = Path(os.environ.get("TF_BUILD_OUT", HERE / "libtomoforge_b200.so"))
OBJ = HERE.parent / "build" / ("obj" + "".join(d.replace("-D", "_").replace("=", "")
                                               for d in _DEFINES))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
]


def units():
    return sorted(CSRC.glob("*.cu"))


def headers():
    return sorted(CSRC.glob("*.cuh"))


def _digest(paths, extra=()) -> str:
    """Content hash of sources + headers + flags: a stale library (or object) is
    rebuilt whatever the file times say (snapshots copied to a GPU box keep or
    reset mtimes arbitrarily)."""
    h = hashlib.sha256()
    for p in paths:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    for e in (*NVCC_FLAGS, *_DEFINES, *extra):
        h.update(e.encode())
    return h.hexdigest()


def _stamp(path: Path) -> Path:
    return path.with_name(path.name + ".sha256")


def library_digest() -> str:
    return _digest(units() + headers())


def up_to_date() -> bool:
    stamp = _stamp(LIB)
    return LIB.exists() and stamp.exists() and stamp.read_text().strip() == library_digest()


def _compile(nvcc: str, src: Path, verbose: bool):
    obj = OBJ / (src.stem + ".o")
    want = _digest([src] + headers())
    if obj.exists() and _stamp(obj).exists() and _stamp(obj).read_text().strip() == want:
        return obj, None
    cmd = [nvcc, *NVCC_FLAGS, *_DEFINES, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        return obj, f"{src.name}: nvcc failed ({res.returncode})\n{res.stdout}{res.stderr}"
    if verbose:
        sys.stderr.write(res.stderr)
    _stamp(obj).write_text(want)
    return obj, None


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    OBJ.mkdir(parents=True, exist_ok=True)
    if force:
        for o in OBJ.glob("*.o"):
            o.unlink()
    with ThreadPoolExecutor(max_workers=len(units())) as ex:
        results = list(ex.map(lambda s: _compile(nvcc, s, verbose), units()))
    errors = [e for _, e in results if e]
    if errors:
        sys.stderr.write("\n".join(errors))
        raise RuntimeError("nvcc failed")
    objs = [str(o) for o, _ in results]
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o",
           str(LIB) + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc link failed ({res.returncode})")
    os.replace(str(LIB) + ".tmp", LIB)
    _stamp(LIB).write_text(library_digest())
    return LIB


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
