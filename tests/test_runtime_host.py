"""Slab runtime host logic: partition rule and the torch.distributed protocol (gloo, CPU)."""

import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import golden
from paper_2603_28756_b200.runtime import SlabPartition, exchange_halos, partition


def test_partition_matches_reference():
    d = golden("runtime.npz")
    for key in ("10_3", "8_4", "7_7", "2048_8", "13_5"):
        n, w = map(int, key.split("_"))
        np.testing.assert_array_equal([[p.begin, p.end] for p in partition(n, w)], d[key])


@pytest.mark.parametrize("n,w", [(1, 1), (5, 2), (17, 4), (64, 8), (2048, 8)])
def test_partition_tiling(n, w):
    parts = partition(n, w)
    assert parts[0].begin == 0 and parts[-1].end == n
    assert all(a.end == b.begin for a, b in zip(parts, parts[1:]))
    sizes = [p.size for p in parts]
    assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    assert parts[0].lower is None and parts[-1].upper is None


def test_partition_errors():
    with pytest.raises(ValueError):
        partition(3, 0)
    with pytest.raises(ValueError):
        partition(3, 4)
    with pytest.raises(ValueError):
        SlabPartition(0, 2, 2, None, None)


def test_exchange_halos_driver_form():
    """test_runtime.py:82-97: each halo is the neighbour's boundary plane."""
    vol = np.arange(6 * 3 * 3, dtype=float).reshape(6, 3, 3)
    parts = partition(6, 3)
    halos = exchange_halos(parts, [vol[p.begin:p.end] for p in parts])
    assert halos[0][0] is None and halos[-1][1] is None
    np.testing.assert_array_equal(halos[1][0], vol[1])
    np.testing.assert_array_equal(halos[1][1], vol[4])
    with pytest.raises(ValueError):
        exchange_halos(parts, [vol[:1], vol[1:3], vol[3:]])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,n_slices", [(2, 5), (3, 7)])
def test_slab_comm_gloo(tmp_path, world, n_slices):
    from _dist_workers import comm_worker

    side = 4
    mp.spawn(comm_worker, args=(world, _free_port(), n_slices, side, str(tmp_path)), nprocs=world,
             join=True)
    full = np.arange(n_slices * side * side, dtype=np.float32).reshape(n_slices, side, side)
    parts = partition(n_slices, world)
    for p in parts:
        r = np.load(tmp_path / f"rank{p.worker_id}.npy", allow_pickle=True).item()
        want_lo = full[p.begin - 1] if p.lower is not None else None
        want_hi = full[p.end] if p.upper is not None else None
        for got, want in ((r["lo"], want_lo), (r["hi"], want_hi)):
            if want is None:
                assert got is None
            else:
                np.testing.assert_array_equal(got, want)
        np.testing.assert_array_equal(r["red"], [world, sum(range(world)), n_slices])
        lo_, hi_ = r["range_lohi"]
        np.testing.assert_array_equal(r["range"], full[lo_:hi_])  # p2p level-change planes
        assert r["halo_msgs"] == (p.lower is not None) + (p.upper is not None)
    r0 = np.load(tmp_path / "rank0.npy", allow_pickle=True).item()
    np.testing.assert_array_equal(r0["gather"], full)
    # the protocol's budget: 2 (W - 1) halo planes per exchange (test_runtime.py:239-250)
    total = sum(np.load(tmp_path / f"rank{p.worker_id}.npy", allow_pickle=True).item()["halo_msgs"]
                for p in parts)
    assert total == 2 * (world - 1)


def test_reference_transport_names_are_accepted():
    """InProcessTransport / SocketTransport exist for drop-in imports and are accepted
    (and ignored) where the reference takes a transport (runtime.py:190-286)."""
    import paper_2603_28756_b200 as tf

    for cls in (tf.InProcessTransport, tf.SocketTransport):
        t = cls(2)
        assert t.n_workers == 2
        t.close()
    with pytest.raises(ValueError):
        tf.InProcessTransport(0)
