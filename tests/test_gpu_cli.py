"""CLI end to end on the GPU: phantom -> project -> mbir equals the library calls."""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_28756_b200 as m

    return m


def test_project_and_mbir_match_library(tf, tmp_path):
    from paper_2603_28756_b200 import cli, fileio

    ph, sn, rc, log = (tmp_path / n for n in ("p.raw", "s.raw", "r.raw", "c.csv"))
    assert cli.main(["phantom", "--kind", "shepp-logan", "--side", "48", "--slices", "2",
                     "--out", str(ph)]) == 0
    assert cli.main(["project", "--input", str(ph), "--angles", "40", "--bins", "64",
                     "--out", str(sn)]) == 0
    (tmp_path / "plan.toml").write_text(
        "[geometry]\nimage_side = 48\n[qggmrf]\nsigma = 0.1\nlambda = 0.01\n"
        "[solver]\nmax_iters = 12\ntol = 1e-300\n")  # L by power iteration (converging run)
    assert cli.main(["mbir", "--sino", str(sn), "--plan", str(tmp_path / "plan.toml"),
                     "--out", str(rc), "--log", str(log), "--export-png",
                     str(tmp_path / "prev.pgm")]) == 0
    sino = fileio.load_array(sn)
    ang = np.linspace(0, np.pi, 40, endpoint=False)
    p = tf.NufftPlan(48, tf.polar_sampling(tf.ScanGeometry(angles=ang, detector_bins=64,
                                                            image_side=48)), 1e-6)
    np.testing.assert_array_equal(sino.data, tf.project_volume(p, fileio.load_array(ph)).data)
    ctx = tf.fidelity_context(p, tf.build_psf(p.sampling, 48), sino)
    ref, recs = tf.solve(ctx, tf.QggmrfParams(sigma=0.1, lam=0.01),
                         tf.SolverConfig(max_iters=12, tol=1e-300), tf.fbp(p, sino))
    got = fileio.load_array(rc)
    np.testing.assert_array_equal(got.data, ref.data)
    # a converging reconstruction, not just CLI == library on diverged numbers
    obj = [r.objective for r in recs]
    assert all(np.isfinite(obj)) and obj[-1] < 0.5 * obj[0]
    truth = fileio.load_array(ph).data
    ncc = float(np.sum(got.data * truth) / np.linalg.norm(got.data) / np.linalg.norm(truth))
    assert ncc > 0.9
    lines = log.read_text().splitlines()
    assert lines[0].startswith("# version=") and lines[1].startswith("iter,objective")
    assert len(lines) == 2 + len(recs)
    assert list(tmp_path.glob("prev_w*.pgm"))


def test_load_slab(tf, tmp_path):
    from paper_2603_28756_b200 import fileio

    vol = tf.Volume(np.random.default_rng(0).standard_normal((6, 8, 8)))
    fileio.save_array(tmp_path / "v.raw", vol)
    slab, head = fileio.load_slab(tmp_path / "v.raw", 2, 5)
    assert head["kind"] == "volume" and tuple(slab.shape) == (3, 8, 8) and slab.is_cuda
    assert rel_l2(slab.double().cpu().numpy(), vol.data[2:5]) < 1e-7
    with pytest.raises(ValueError):
        fileio.load_slab(tmp_path / "v.raw", 4, 9)
