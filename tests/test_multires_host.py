"""Host-side multires pieces vs reference fixtures (CPU only)."""

import numpy as np
import pytest

from conftest import golden
from paper_2603_28756_b200.geometry import Sinogram
from paper_2603_28756_b200.multires import (
    GridHierarchy,
    default_hierarchy,
    downsample_sinogram,
    lanczos_kernel,
    lanczos_matrix,
)


def test_lanczos_and_matrices_match_reference():
    d = golden("multires.npz")
    np.testing.assert_array_equal(lanczos_kernel(np.linspace(-4, 4, 81)), d["lanczos"])
    np.testing.assert_allclose(lanczos_matrix(10, 20), d["mat"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(lanczos_matrix(7, 16), d["mat_odd"], rtol=0, atol=1e-15)


def test_downsample_matches_reference():
    d = golden("multires.npz")
    ang = np.linspace(0.0, np.pi, 7, endpoint=False)
    s = Sinogram(angles=ang, data=d["sino"])
    ds = downsample_sinogram(s, 4)
    np.testing.assert_array_equal(ds.data, d["ds_data"])
    np.testing.assert_array_equal(ds.angles, d["ds_angles"])
    np.testing.assert_array_equal(downsample_sinogram(s, 2, downsample_angles=True).data, d["ds_ang"])
    assert downsample_sinogram(s, 1) is s
    with pytest.raises(ValueError):
        downsample_sinogram(s, 3)


def test_stride_rule():
    """test_multires.py:35-42: bins [1, 2, 3, 4] at factor 2 -> [0.5, 1.5]."""
    s = Sinogram(angles=np.array([0.0]), data=np.array([[[1.0, 2.0, 3.0, 4.0]]]))
    np.testing.assert_array_equal(downsample_sinogram(s, 2).data[0, 0], [0.5, 1.5])


def test_band_extraction_reproduces_dense_matrix():
    for n_src, n_tgt in [(10, 20), (7, 16), (1024, 2048), (5, 5), (3, 12)]:
        mat = lanczos_matrix(n_src, n_tgt)
        nz = mat != 0.0
        first = np.argmax(nz, axis=1)
        last = n_src - 1 - np.argmax(nz[:, ::-1], axis=1)
        taps = int((last - first).max()) + 1
        assert taps <= 8
        start = np.minimum(first, n_src - taps)
        idx = start[:, None] + np.arange(taps)[None]
        w = np.take_along_axis(mat, idx, axis=1)
        x = np.random.default_rng(0).standard_normal(n_src)
        np.testing.assert_allclose((w * x[idx]).sum(1), mat @ x, rtol=1e-13, atol=1e-13)


def test_hierarchy_rules():
    h = GridHierarchy(levels=(512, 1024, 2048), iters_per_level=(40, 20, 10))
    assert h.levels[-1] == 2048
    with pytest.raises(ValueError):
        GridHierarchy(levels=(500, 2048), iters_per_level=(1, 1))
    with pytest.raises(ValueError):
        GridHierarchy(levels=(1024, 2048), iters_per_level=(1,))
    d = default_hierarchy(256)
    assert d.levels == (64, 128, 256) and d.iters_per_level == (200, 100, 50)
    assert default_hierarchy(2048, 3, finest_iters=10).iters_per_level == (40, 20, 10)


def test_clear_caches_is_exported():
    import paper_2603_28756_b200 as tf

    tf.clear_caches()  # no device work: only drops dictionary entries
