"""The reference's bench categories on the GPU (paper_2603_28756_b200.benchmarks, the
`bench` CLI subcommand) against CSV files the reference itself wrote
(tests/golden/make_golden.py --only-bench): same columns and metadata keys, the same
config hash where the metadata is the configuration, and the same numbers to fp32
tolerances."""

import csv

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bm():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_28756_b200 import benchmarks

    return benchmarks


def _read(path):
    lines = open(path).read().splitlines()
    meta = dict(kv.split("=", 1) for kv in lines[0][2:].split(" ") if "=" in kv)
    rows = list(csv.reader(lines[1:]))
    return meta, rows[0], rows[1:]


def test_bench_toeplitz_matches_reference_file(bm, tmp_path):
    """Direct projection pair vs Toeplitz gradient (the paper's Fig. 2 comparison)."""
    out = tmp_path / "t.csv"
    bm.bench_toeplitz(out, sizes=(32, 48), n_angles=20, seed=0, repeats=1)
    meta, cols, rows = _read(out)
    rmeta, rcols, rrows = _read(GOLDEN / "bench" / "toeplitz.csv")
    assert cols == rcols and [r[0] for r in rows] == [r[0] for r in rrows]
    assert meta["config_hash"] == rmeta["config_hash"]
    assert set(rmeta) <= set(meta)
    for r in rows:  # the two routes agree to fp32 on the GPU, as to fp64 in the reference
        assert float(r[3]) < 1e-5 and float(r[4]) < 1e-4
        assert float(r[1]) > 0 and float(r[2]) > 0


def test_bench_init_matches_reference_file(bm, tmp_path):
    out = tmp_path / "i.csv"
    curves = bm.bench_init(out, side=64, n_angles=30, max_iters=20, seed=7)
    meta, cols, rows = _read(out)
    rmeta, rcols, rrows = _read(GOLDEN / "bench" / "init.csv")
    assert cols == rcols and len(rows) == len(rrows)
    assert float(meta["sigma"]) == pytest.approx(float(rmeta["sigma"]), rel=1e-4)
    assert [(r[0], r[1], r[4]) for r in rows] == [(r[0], r[1], r[4]) for r in rrows]
    got = np.array([[float(r[2]), float(r[3])] for r in rows])
    ref = np.array([[float(r[2]), float(r[3])] for r in rrows])
    np.testing.assert_allclose(got, ref, rtol=1e-4)
    assert curves["fbp"][0].fidelity < curves["zero"][0].fidelity


def test_bench_multires_matches_reference_file(bm, tmp_path):
    out = tmp_path / "m.csv"
    res = bm.bench_multires(out, side=64, n_angles=30, single_iters=40, fine_iters=8, seed=7)
    meta, cols, rows = _read(out)
    rmeta, rcols, rrows = _read(GOLDEN / "bench" / "multires.csv")
    assert cols == rcols and [r[:3] for r in rows] == [r[:3] for r in rrows]
    got = np.array([[float(r[3]), float(r[4])] for r in rows])
    ref = np.array([[float(r[3]), float(r[4])] for r in rrows])
    # noise-free, lam = 0: the residual falls towards the fp32 floor, so the tolerance
    # is relative to the run's starting residual once the values get small
    np.testing.assert_allclose(got, ref, rtol=1e-3, atol=1e-5 * ref[0, 0])
    assert res["t_single"] > 0 and res["t_multi"] > 0


def test_bench_scaling_runs_worker_processes(bm, tmp_path):
    """W = 1 in-process and W = 2 as two slab processes (gloo on one GPU here)."""
    out = tmp_path / "s.csv"
    times = bm.bench_scaling(out, workers=(1, 2), side=32, slices=8, iters=2, seed=3)
    meta, cols, rows = _read(out)
    assert cols == ["workers", "wall_s"] and [r[0] for r in rows] == ["1", "2"]
    assert all(t > 0 for t in times.values())


def test_cli_bench_toeplitz(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_28756_b200 import cli

    out = tmp_path / "c.csv"
    assert cli.main(["bench", "toeplitz", "--out", str(out), "--sizes", "32", "--angles",
                     "20"]) == 0
    _, cols, rows = _read(out)
    assert cols[0] == "N" and rows[0][0] == "32"
