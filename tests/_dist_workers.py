"""Multi-process workers for the runtime tests (spawned with torch.multiprocessing)."""

import os

import numpy as np
import torch
import torch.distributed as dist


def _init(rank, world, port, backend="gloo"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)


def comm_worker(rank, world, port, n_slices, side, out_dir):
    """Exchange / allreduce / gather of the slab protocol on CPU tensors (gloo)."""
    from paper_2603_28756_b200.runtime import SlabComm, partition

    _init(rank, world, port)
    try:
        parts = partition(n_slices, world)
        part = parts[rank]
        full = np.arange(n_slices * side * side, dtype=np.float32).reshape(n_slices, side, side)
        slab = torch.from_numpy(full[part.begin:part.end].copy())
        comm = SlabComm(part)
        lo, hi = comm.exchange(slab)
        red = comm.allreduce(torch.tensor([1.0, float(rank), float(part.size)], dtype=torch.float64))
        g = comm.gather(slab, parts)
        # level-change transfer: rank r needs planes [r, n_slices - world + r + 1) (overlapping
        # ranges of different lengths, crossing several slabs)
        ranges = [(q, n_slices - world + q + 1) for q in range(world)]
        rng_planes = comm.gather_range(slab, parts, ranges)
        res = {"lo": None if lo is None else lo.numpy(), "hi": None if hi is None else hi.numpy(),
               "red": red.numpy(), "halo_msgs": comm.counts["halo"],
               "range": rng_planes.numpy(), "range_lohi": ranges[rank]}
        if rank == 0:
            res["gather"] = g.numpy()
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def solve_worker(rank, world, port, fixture, out_dir):
    """distributed_solve on cuda:0 with a gloo group (host-staged halos)."""
    import paper_2603_28756_b200 as tf
    from paper_2603_28756_b200.runtime import distributed_solve

    torch.cuda.set_device(0)
    _init(rank, world, port)
    try:
        d = dict(np.load(fixture))
        sino = tf.Sinogram(angles=d["angles"], data=d["g"])
        prm = tf.QggmrfParams(sigma=0.3, lam=0.05)
        cfg = tf.SolverConfig(max_iters=8, tol=1e-300, lipschitz=None)
        snaps = []
        vol, recs = distributed_solve(sino, 16, prm, cfg, world,
                                      snapshot_sink=lambda k, v: snaps.append(v))
        # the same solve from a saved sinogram: each rank memory-maps its own rows
        from paper_2603_28756_b200 import fileio

        path = os.path.join(out_dir, "sino.raw")
        if rank == 0:
            fileio.save_array(path, sino)
        dist.barrier()
        vol_p, _ = distributed_solve(path, 16, prm, cfg, world)
        if rank == 0:
            np.save(os.path.join(out_dir, "solve.npy"),
                    {"vol": vol.data, "obj": np.array([r.objective for r in recs]),
                     "nsnap": len(snaps), "vol_path": vol_p.data}, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def solve7_worker(rank, world, port, out_dir):
    """7-slice problem (24^2, 12 angles) on cuda:0; W = world over gloo (W = 1: no group)."""
    import paper_2603_28756_b200 as tf
    from paper_2603_28756_b200.runtime import distributed_solve

    torch.cuda.set_device(0)
    if world > 1:
        _init(rank, world, port)
    try:
        ang = np.linspace(0, np.pi, 12, endpoint=False)
        g = np.random.default_rng(7).standard_normal((7, 12, 24))
        sino = tf.Sinogram(angles=ang, data=g)
        prm = tf.QggmrfParams(sigma=0.3, lam=0.05)
        cfg = tf.SolverConfig(max_iters=6, tol=1e-300, lipschitz=300.0)
        vol, recs = distributed_solve(sino, 24, prm, cfg, world)
        if rank == 0:
            np.save(os.path.join(out_dir, f"solve7_w{world}.npy"),
                    {"vol": vol.data, "obj": np.array([r.objective for r in recs])},
                    allow_pickle=True)
    finally:
        if world > 1:
            dist.destroy_process_group()


def hier_worker(rank, world, port, fixture, out_dir):
    """distributed_solve_hierarchical on cuda:0 (gloo) for the hier.npz problem."""
    import paper_2603_28756_b200 as tf
    from paper_2603_28756_b200.runtime import distributed_solve_hierarchical

    torch.cuda.set_device(0)
    _init(rank, world, port)
    try:
        d = dict(np.load(fixture))
        sino = tf.Sinogram(angles=d["angles"], data=d["g"])
        prm = tf.QggmrfParams(sigma=0.1, lam=1e-2)
        hier = tf.GridHierarchy(levels=(16, 32), iters_per_level=(6, 4))
        vol, lrecs = distributed_solve_hierarchical(sino, hier, prm,
                                                    tf.SolverConfig(max_iters=1, tol=1e-300),
                                                    world, use_fbp_init=True)
        if rank == 0:
            np.save(os.path.join(out_dir, "hier.npy"),
                    {"vol": vol.data, "obj0": np.array([r.objective for r in lrecs[0]]),
                     "obj1": np.array([r.objective for r in lrecs[1]])}, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def diverge_worker(rank, world, port, fixture, out_dir):
    """distributed_solve with a far too small Lipschitz constant: must raise
    RuntimeError('worker <rank> failed: ...') wrapping the FloatingPointError."""
    import paper_2603_28756_b200 as tf
    from paper_2603_28756_b200.runtime import distributed_solve

    torch.cuda.set_device(0)
    _init(rank, world, port)
    try:
        d = dict(np.load(fixture))
        sino = tf.Sinogram(angles=d["angles"], data=d["g"])
        prm = tf.QggmrfParams(sigma=0.3, lam=0.05)
        cfg = tf.SolverConfig(max_iters=500, tol=1e-300, lipschitz=1e-6, restart=False)
        try:
            distributed_solve(sino, 16, prm, cfg, world)
            msg = "no error"
        except Exception as exc:  # noqa: BLE001 - recorded for the test
            msg = f"{type(exc).__name__}: {exc}"
        with open(os.path.join(out_dir, f"diverge{rank}.txt"), "w") as fh:
            fh.write(msg)
    finally:
        dist.destroy_process_group()


def peer_halo_worker(rank, world, port, out_dir):
    """distributed_solve (3-D, 9 slices over `world` ranks on cuda:0, gloo control plane)
    with the halo planes sent over the group ("nccl" path: host-staged on gloo) and
    written into the neighbours' IPC-mapped inboxes ("peer"); plus the hierarchical
    solve with peer halos."""
    import paper_2603_28756_b200 as tf
    from paper_2603_28756_b200.runtime import distributed_solve, distributed_solve_hierarchical

    torch.cuda.set_device(0)
    _init(rank, world, port)
    try:
        ang = np.linspace(0, np.pi, 12, endpoint=False)
        g = np.random.default_rng(9).standard_normal((9, 12, 24))
        sino = tf.Sinogram(angles=ang, data=g)
        prm = tf.QggmrfParams(sigma=0.3, lam=0.05)
        cfg = tf.SolverConfig(max_iters=7, tol=1e-300, lipschitz=300.0)
        res = {}
        for halo in ("nccl", "peer"):
            vol, recs = distributed_solve(sino, 24, prm, cfg, world, halo=halo)
            if rank == 0:
                res[halo] = (vol.data, np.array([r.objective for r in recs]))
        hier = tf.GridHierarchy(levels=(12, 24), iters_per_level=(4, 3))
        for halo in ("nccl", "peer"):
            vol, lrecs = distributed_solve_hierarchical(
                sino, hier, prm, tf.SolverConfig(max_iters=1, tol=1e-300), world,
                use_fbp_init=True, halo=halo)
            if rank == 0:
                res["hier_" + halo] = (vol.data, np.array([r.objective for r in lrecs[-1]]))
        if rank == 0:
            np.save(os.path.join(out_dir, f"peer_w{world}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()
