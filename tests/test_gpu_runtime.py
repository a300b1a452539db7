"""distributed_solve on the GPU: W=1 and W=2 (two processes on cuda:0, gloo group,
host-staged halos) against the reference's single- and two-worker runs."""

import socket

import numpy as np
import pytest

from conftest import GOLDEN, golden, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_28756_b200 as m

    return m


def test_single_worker_matches_reference(tf):
    from paper_2603_28756_b200.runtime import distributed_solve

    d = golden("runtime.npz")
    sino = tf.Sinogram(angles=d["angles"], data=d["g"])
    prm = tf.QggmrfParams(sigma=0.3, lam=0.05)
    vol, recs = distributed_solve(sino, 16, prm, tf.SolverConfig(max_iters=8, tol=1e-300), 1)
    assert rel_l2(vol.data, d["recon_w1"]) < 1e-3
    np.testing.assert_allclose([r.objective for r in recs], d["obj_w1"], rtol=1e-4)


def test_two_workers_match_single_worker(tf, tmp_path):
    import torch.multiprocessing as mp

    from _dist_workers import solve_worker

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(solve_worker, args=(2, port, str(GOLDEN / "runtime.npz"), str(tmp_path)), nprocs=2,
             join=True)
    r = np.load(tmp_path / "solve.npy", allow_pickle=True).item()
    d = golden("runtime.npz")
    # the reference's own W=2 run equals its W=1 run; ours must match both
    assert rel_l2(r["vol"], d["recon_w2"]) < 1e-3
    np.testing.assert_allclose(r["obj"], d["obj_w2"], rtol=1e-4)
    assert r["nsnap"] == 8
    np.testing.assert_array_equal(r["vol_path"], r["vol"])  # sinogram read per rank from a file


def test_worker_count_must_match_group(tf):
    from paper_2603_28756_b200.runtime import distributed_solve

    d = golden("runtime.npz")
    sino = tf.Sinogram(angles=d["angles"], data=d["g"])
    with pytest.raises(ValueError):
        distributed_solve(sino, 16, tf.QggmrfParams(sigma=0.3), tf.SolverConfig(max_iters=1), 2)
    with pytest.raises(ValueError):
        distributed_solve(sino, 16, tf.QggmrfParams(sigma=0.3), tf.SolverConfig(max_iters=1), 7)


def test_hierarchical_over_slabs_matches_reference(tf, tmp_path):
    """Multires x z-slabs (W = 2 on one GPU) against the reference's single-worker
    hierarchical run (hier.npz): levels (16, 32), FBP init, 2 -> 4 slices."""
    import torch.multiprocessing as mp

    from _dist_workers import hier_worker

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(hier_worker, args=(2, port, str(GOLDEN / "hier.npz"), str(tmp_path)), nprocs=2,
             join=True)
    r = np.load(tmp_path / "hier.npy", allow_pickle=True).item()
    d = golden("hier.npz")
    assert rel_l2(r["vol"], d["recon"]) < 1e-3
    np.testing.assert_allclose(r["obj0"], d["obj0"], rtol=1e-4)
    np.testing.assert_allclose(r["obj1"], d["obj1"], rtol=1e-4)


def test_worker_divergence_is_runtime_error(tf, tmp_path):
    """A diverging slab solve surfaces as RuntimeError('worker i failed ...') on every
    rank, as the reference's threads do (runtime.py:684-690; its
    test_worker_failure_propagates)."""
    import torch.multiprocessing as mp

    from _dist_workers import diverge_worker

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(diverge_worker, args=(2, port, str(GOLDEN / "runtime.npz"), str(tmp_path)),
             nprocs=2, join=True)
    for rank in range(2):
        msg = (tmp_path / f"diverge{rank}.txt").read_text()
        assert msg.startswith("RuntimeError") and "worker" in msg and "non-finite" in msg


@pytest.mark.parametrize("world", [2, 3])
def test_peer_memory_halos_match_group_halos(tf, tmp_path, world):
    """halo="peer" (planes copied into the neighbours' IPC-mapped inboxes, flag
    published / awaited by tf_halo_signal / tf_halo_wait) gives bit-for-bit the
    reconstruction of the group send/recv path, for plain and hierarchical solves."""
    import torch.multiprocessing as mp

    from _dist_workers import peer_halo_worker

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(peer_halo_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    r = np.load(tmp_path / f"peer_w{world}.npy", allow_pickle=True).item()
    for a, b in (("nccl", "peer"), ("hier_nccl", "hier_peer")):
        np.testing.assert_array_equal(r[a][0], r[b][0])
        np.testing.assert_array_equal(r[a][1], r[b][1])
