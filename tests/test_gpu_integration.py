"""INTEGRATION.md's reference-side ctypes stub, executed verbatim (extracted from the
markdown) against the reference-generated Toeplitz fixtures: the binding a tomoforge
maintainer would add is exercised, not just documented."""

import glob
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, rel_l2

pytestmark = pytest.mark.gpu


def _stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    block = text.split("<!-- stub:begin -->", 1)[1].split("<!-- stub:end -->", 1)[0]
    return re.search(r"```python\n(.*?)```", block, re.S).group(1)


@pytest.fixture(scope="module")
def stub():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_28756_b200 import _lib

    os.environ["TOMOFORGE_B200_LIB"] = str(_lib.LIB_PATH)
    ns = {"__name__": "tomoforge._b200"}
    exec(compile(_stub_source(), "INTEGRATION.md:stub", "exec"), ns)  # noqa: S102
    return ns


@pytest.mark.parametrize("path", sorted(glob.glob(str(GOLDEN / "toeplitz_*.npz"))),
                         ids=lambda p: os.path.basename(p))
def test_stub_apply_and_gradient(stub, path):
    d = dict(np.load(path))
    side = int(d["f"].shape[-1])
    psf = stub["B200Psf"](d["angles"], d["g"].shape[-1], side)
    assert psf.M >= 2 * side - 1
    assert rel_l2(stub["apply_batch"](psf, d["f"]), d["kf"]) < 1e-5
    grad = stub["apply_batch"](psf, d["f"], aux=d["rstar"], beta=-1.0)
    assert rel_l2(grad, d["grad"]) < 1e-4


def test_stub_maps_errors(stub):
    """-1 from the library (here: a side above the supported maximum) is ValueError."""
    with pytest.raises(ValueError, match="unsupported|side|bad"):
        stub["B200Psf"](np.linspace(0, np.pi, 6, endpoint=False), 16, 5000)
