"""z-slab parallel MBIR: one process per GPU, NCCL halo exchange + scalar allreduce.

Drop-in for the slab runtime of tomoforge/runtime.py: ``SlabPartition`` /
``partition`` (runtime.py:82-125), ``exchange_halos`` (:345-367) and
``distributed_solve`` (:622-691) with the worker loop of :523-619.

The reference runs one thread per slab and models MPI with queue/socket
transports.  Here every slab is a process bound to one GPU (torchrun), and the
protocol is carried by ``torch.distributed``:

* per iteration exactly one halo exchange: each rank sends its first plane of
  the new iterate to the lower neighbour and its last plane to the upper one
  (contiguous N^2 fp32 planes -- no packing), 2 (W-1) messages in total,
  NCCL send/recv straight from device memory (``batch_isend_irecv``); on a
  gloo group the planes are staged through host memory;
* one allreduce of three fp64 scalars [energy, fidelity increment, ||grad||^2],
  so every rank takes the identical restart / stop decision
  (runtime.py:581-588; the sum is bitwise identical on all ranks);
* the extrapolated point's halos are never sent: the fused K4 kernel forms
  y = f + c (f - f_prev) on the fly, halo planes included (runtime.py:590-597);
* the fidelity term is slice-local, so the Toeplitz apply and R*g need no
  communication (runtime.py:5-6).

The objective bookkeeping is the single-GPU solver's (solver.py): increments
accumulated in fp64 and reduced across ranks.
"""

from __future__ import annotations

import collections
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _lib
from .geometry import ScanGeometry, Sinogram, Volume, polar_sampling
from .nufft import NufftPlan
from .qggmrf import stencil_2d, stencil_3d
from .radon import back_project_stack
from .solver import SolverConfig, _iterate, estimate_lipschitz, solve
from .toeplitz import FidelityContext, build_psf, fidelity_context

__all__ = [
    "SlabPartition",
    "TransportError",
    "ProtocolError",
    "TransportTimeout",
    "SlabComm",
    "partition",
    "exchange_halos",
    "distributed_solve",
    "distributed_solve_hierarchical",
    "InProcessTransport",
    "SocketTransport",
]


class TransportError(RuntimeError):
    pass


class ProtocolError(TransportError):
    """A slab or plane does not match the partition it is exchanged under."""


class TransportTimeout(TransportError):
    """An expected neighbour message never arrived (collective timeout)."""


class _TransportMarker:
    """Name-compatible stand-in for the reference's CPU transports (runtime.py:190-286).

    The reference models MPI with in-process queues or local sockets between worker
    threads; here the slab workers are GPU processes and the transport is the
    torch.distributed group (NCCL, or gloo for tests), plus optional peer-memory
    halos (``halo="peer"``).  Instances are accepted wherever the reference takes a
    ``transport`` argument and are otherwise inert: the queue / socket protocol itself
    is out of scope."""

    def __init__(self, n_workers: int, *args, **kwargs):
        if n_workers < 1:
            raise ValueError("need at least one worker")
        self.n_workers = n_workers

    def close(self):
        pass


class InProcessTransport(_TransportMarker):
    __doc__ = _TransportMarker.__doc__


class SocketTransport(_TransportMarker):
    __doc__ = _TransportMarker.__doc__


@dataclass(frozen=True)
class SlabPartition:
    """Contiguous slice range [begin, end) owned by one worker (runtime.py:82-105)."""

    worker_id: int
    begin: int
    end: int
    lower: int | None
    upper: int | None
    halo_width: int = 1

    def __post_init__(self):
        if self.end <= self.begin:
            raise ValueError("empty slab")
        if self.halo_width != 1:
            raise ValueError("halo width is fixed at 1 (26-neighbor stencil reach)")

    @property
    def slice_range(self):
        return (self.begin, self.end)

    @property
    def size(self) -> int:
        return self.end - self.begin


def partition(n_slices: int, n_workers: int) -> list[SlabPartition]:
    """Balanced contiguous slabs, sizes differ by at most 1, larger first (runtime.py:108-125)."""
    if n_workers < 1:
        raise ValueError("need at least one worker")
    if n_slices < n_workers:
        raise ValueError(f"cannot split {n_slices} slices across {n_workers} workers")
    base, extra = divmod(n_slices, n_workers)
    parts, begin = [], 0
    for w in range(n_workers):
        size = base + (1 if w < extra else 0)
        parts.append(SlabPartition(worker_id=w, begin=begin, end=begin + size,
                                   lower=w - 1 if w > 0 else None,
                                   upper=w + 1 if w < n_workers - 1 else None))
        begin += size
    return parts


def exchange_halos(partitions, slabs, iteration: int = 0, transport=None):
    """Driver-side bulk exchange over all slabs held by one process (runtime.py:345-367):
    one ``(halo_lo, halo_hi)`` per slab, ``None`` on open ends.  The lower halo is
    the lower neighbour's last plane, the upper halo the upper neighbour's first."""
    if len(partitions) != len(slabs):
        raise ValueError("need exactly one slab per partition")
    for part, slab in zip(partitions, slabs):
        if slab.shape[0] != part.size:
            raise ValueError(f"slab of worker {part.worker_id} has {slab.shape[0]} slices, "
                             f"expected {part.size}")
    out = []
    for part in partitions:
        lo = slabs[part.lower][-1] if part.lower is not None else None
        hi = slabs[part.upper][0] if part.upper is not None else None
        out.append((lo, hi))
    return out


class SlabComm:
    """This rank's end of the slab protocol over a torch.distributed group.

    ``exchange(slab)`` returns the (lower, upper) halo planes of ``slab`` (None on
    open ends); ``allreduce(values)`` sums a short fp64 vector.  ``counts`` keeps
    per-purpose message counts (the reference's protocol budget,
    test_runtime.py:239-250).
    """

    def __init__(self, part: SlabPartition, group=None, halo: str = "nccl"):
        self.part = part
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.rank != part.worker_id:
            raise ProtocolError(f"rank {self.rank} given the partition of worker {part.worker_id}")
        if halo not in ("nccl", "peer"):
            raise ValueError("halo must be 'nccl' or 'peer'")
        self.direct = dist.get_backend(group) == "nccl"
        self.halo = halo
        self._peer_halo = None  # _PeerHalo, created at the first exchange (plane shape known)
        self.counts = collections.Counter()

    def _peer(self, w):
        return w if self.group is None else dist.get_global_rank(self.group, w)

    def exchange(self, slab: torch.Tensor):
        return self.exchange_finish(self.exchange_start(slab))

    def exchange_start(self, slab: torch.Tensor):
        """Post the boundary-plane sends/receives of ``slab``.  With NCCL and device
        tensors the transfers run on NCCL's stream while the caller keeps
        launching work (the solver overlaps them with the slab's Toeplitz
        apply); ``exchange_finish`` makes the current stream wait for them."""
        part = self.part
        if slab.shape[0] != part.size:
            raise ProtocolError(f"slab has {slab.shape[0]} slices, partition owns {part.size}")
        if self.halo == "peer" and slab.is_cuda:
            if self._peer_halo is None:
                self._peer_halo = _PeerHalo(self, tuple(slab.shape[1:]), slab.dtype, slab.device)
            self.counts["halo"] += (part.lower is not None) + (part.upper is not None)
            return self._peer_halo.start(slab)
        plane_shape = slab.shape[1:]
        staged = not (self.direct and slab.is_cuda)
        buf_dev = "cpu" if staged else slab.device
        ops, lo, hi = [], None, None

        def out(t):
            return t.to("cpu") if staged else t

        if part.lower is not None:
            lo = torch.empty(plane_shape, dtype=slab.dtype, device=buf_dev)
            ops.append(dist.P2POp(dist.isend, out(slab[0]).contiguous(), self._peer(part.lower),
                                  self.group))
            ops.append(dist.P2POp(dist.irecv, lo, self._peer(part.lower), self.group))
            self.counts["halo"] += 1
        if part.upper is not None:
            hi = torch.empty(plane_shape, dtype=slab.dtype, device=buf_dev)
            ops.append(dist.P2POp(dist.isend, out(slab[-1]).contiguous(), self._peer(part.upper),
                                  self.group))
            ops.append(dist.P2POp(dist.irecv, hi, self._peer(part.upper), self.group))
            self.counts["halo"] += 1
        reqs = dist.batch_isend_irecv(ops) if ops else []
        if staged:  # host-staged (gloo): complete now
            for req in reqs:
                req.wait()
            reqs = []
            if slab.is_cuda:
                lo = lo.to(slab.device) if lo is not None else None
                hi = hi.to(slab.device) if hi is not None else None
        return reqs, lo, hi

    def exchange_finish(self, handle):
        if isinstance(handle, _PeerTicket):
            return self._peer_halo.finish(handle)
        reqs, lo, hi = handle
        for req in reqs:
            req.wait()
        return lo, hi

    def allreduce(self, values: torch.Tensor) -> torch.Tensor:
        """Sum of an fp64 vector over the group (identical on every rank)."""
        t = values.to(torch.float64)
        if not (self.direct and t.is_cuda):
            t = t.cpu()
        t = t.clone()
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        self.counts["reduce"] += 1
        return t

    def broadcast_scalar(self, value: float | None, root: int = 0) -> float:
        dev = torch.device("cuda", torch.cuda.current_device()) if self.direct else "cpu"
        t = torch.tensor([value if value is not None else 0.0], dtype=torch.float64, device=dev)
        dist.broadcast(t, src=self._peer(root), group=self.group)
        return float(t.item())

    def allgather(self, slab: torch.Tensor, parts) -> torch.Tensor:
        """The full volume on every rank (slabs padded to the largest size)."""
        big = max(p.size for p in parts)
        dev = slab.device if (self.direct and slab.is_cuda) else torch.device("cpu")
        pad = torch.zeros((big,) + tuple(slab.shape[1:]), dtype=slab.dtype, device=dev)
        pad[:slab.shape[0]] = slab.to(dev)
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(bufs, pad, group=self.group)
        self.counts["allgather"] += 1
        full = torch.cat([bufs[p.worker_id][:p.size] for p in parts])
        return full.to(slab.device)

    def gather_range(self, slab: torch.Tensor, parts, ranges):
        """Planes [lo, hi) = ``ranges[self.rank]`` of the volume distributed as ``parts``,
        by point-to-point transfers of only the overlapping planes (every rank knows
        every rank's range).  Replaces a whole-volume all-gather at a level change:
        a fine slab's Lanczos z-taps need its own coarse planes +-3."""
        me = parts[self.rank]
        lo, hi = ranges[self.rank]
        staged = not (self.direct and slab.is_cuda)
        dev = torch.device("cpu") if staged else slab.device
        out = torch.empty((hi - lo,) + tuple(slab.shape[1:]), dtype=slab.dtype, device=dev)
        src = slab.to(dev) if staged else slab
        ops = []
        for q, (qlo, qhi) in enumerate(ranges):  # what I send to q
            a, b = max(me.begin, qlo), min(me.end, qhi)
            if a >= b:
                continue
            if q == self.rank:
                out[a - lo:b - lo] = src[a - me.begin:b - me.begin]
            else:
                ops.append(dist.P2POp(dist.isend, src[a - me.begin:b - me.begin].contiguous(),
                                      self._peer(q), self.group))
        for q, p in enumerate(parts):  # what I receive from q
            a, b = max(p.begin, lo), min(p.end, hi)
            if a >= b or q == self.rank:
                continue
            ops.append(dist.P2POp(dist.irecv, out[a - lo:b - lo], self._peer(q), self.group))
        for req in (dist.batch_isend_irecv(ops) if ops else []):
            req.wait()
        self.counts["range"] += 1
        return out.to(slab.device)

    def gather(self, slab: torch.Tensor, parts, root: int = 0):
        """Full volume on ``root`` (None elsewhere); slabs padded to the largest size."""
        big = max(p.size for p in parts)
        dev = slab.device if (self.direct and slab.is_cuda) else torch.device("cpu")
        pad = torch.zeros((big,) + tuple(slab.shape[1:]), dtype=slab.dtype, device=dev)
        pad[:slab.shape[0]] = slab.to(dev)
        bufs = [torch.empty_like(pad) for _ in range(self.world)] if self.rank == root else None
        dist.gather(pad, bufs, dst=self._peer(root), group=self.group)
        self.counts["gather"] += 1
        if self.rank != root:
            return None
        return torch.cat([bufs[p.worker_id][:p.size] for p in parts])


@dataclass(frozen=True)
class _PeerTicket:
    parity: int
    value: int


class _PeerHalo:
    """Halo planes written straight into the neighbours' device memory (csrc/halo.cu).

    Each rank's inbox -- [parity][lo, hi] planes plus a uint64 flag per slot -- is
    shared once over the group (CUDA IPC handles, all_gather_object) and mapped by
    the neighbours, over NVLink when they are other GPUs of the node.  ``start``
    copies this slab's first / last plane into the lower / upper neighbour's slot
    (stream-ordered peer copies) and publishes the exchange number there
    (tf_halo_signal); ``finish`` makes the stream wait for both neighbours' flags
    (tf_halo_wait) and returns views of its own inbox.  Two parity slots suffice
    because the per-iteration scalar allreduce keeps the ranks in lockstep."""

    def __init__(self, comm: "SlabComm", plane_shape, dtype, device):
        from torch.multiprocessing.reductions import reduce_tensor

        self.comm, self.part = comm, comm.part
        self.inbox = torch.zeros((2, 2) + tuple(plane_shape), dtype=dtype, device=device)
        self.flags = torch.zeros((2, 2), dtype=torch.int64, device=device)
        mine = (reduce_tensor(self.inbox), reduce_tensor(self.flags))
        objs = [None] * comm.world
        dist.all_gather_object(objs, mine, group=comm.group)
        self.peer = {}
        for q in (self.part.lower, self.part.upper):
            if q is not None:
                (f_in, a_in), (f_fl, a_fl) = objs[q]
                self.peer[q] = (f_in(*a_in), f_fl(*a_fl))
        self.count = 0

    def start(self, slab: torch.Tensor) -> _PeerTicket:
        lib = _lib.ensure_ready()
        k = self.count
        self.count += 1
        p, value = k & 1, k + 1
        st = _lib.stream_handle()
        for q, plane, side in ((self.part.lower, slab[0], 1), (self.part.upper, slab[-1], 0)):
            if q is None:
                continue
            inbox, flags = self.peer[q]
            inbox[p, side].copy_(plane, non_blocking=True)  # my boundary = q's halo
            _lib.check(lib.tf_halo_signal(flags[p, side].data_ptr(), value, st),
                       "tf_halo_signal")
        return _PeerTicket(p, value)

    def finish(self, t: _PeerTicket):
        lib = _lib.ensure_ready()
        lo_ok, hi_ok = self.part.lower is not None, self.part.upper is not None
        _lib.check(lib.tf_halo_wait(self.flags[t.parity, 0].data_ptr() if lo_ok else None,
                                    self.flags[t.parity, 1].data_ptr() if hi_ok else None,
                                    t.value, _lib.stream_handle()), "tf_halo_wait")
        return (self.inbox[t.parity, 0] if lo_ok else None,
                self.inbox[t.parity, 1] if hi_ok else None)


class _Rows:
    """The sinogram a slab solve reads from: a ``Sinogram``, or the path of a saved
    one (fileio format), memory-mapped so that each rank touches only its own rows
    (a 2048^3 scan is 4.3 GB of float64 per process otherwise)."""

    def __init__(self, sino):
        if isinstance(sino, Sinogram):
            self.angles, self._data = sino.angles, sino.data
            return
        from . import fileio

        path = __import__("pathlib").Path(sino)
        head = fileio._read_header(path)
        if head["kind"] != "sinogram":
            raise ValueError(f"{path} holds a {head['kind']}, not a sinogram")
        self.angles = np.asarray(head["angles"], dtype=np.float64)
        self._data = np.memmap(path, dtype="<f8", mode="r", shape=tuple(head["dims"]))

    slices = property(lambda self: self._data.shape[0])
    detector_bins = property(lambda self: self._data.shape[2])

    def rows(self, idx) -> np.ndarray:
        """float64 rows of slices ``idx`` (a slice or index array): only those are read."""
        return np.asarray(self._data[idx], dtype=np.float64)

    def sinogram(self) -> Sinogram:
        return Sinogram(angles=self.angles, data=self.rows(slice(None)))


def distributed_solve(sino: Sinogram, image_side: int, params, cfg: SolverConfig, n_workers: int,
                      *, f0: Volume | None = None, transport=None, nufft_tolerance: float = 1e-6,
                      oversampling: float = 2.0, on_record=None, snapshot_sink=None,
                      gather: str = "root", group=None, halo: str = "nccl"):
    """Slab-parallel reconstruction, algebraically identical to ``solve`` (runtime.py:622-691).

    SPMD: every rank of the process group (one per GPU, ``n_workers`` = group
    size) calls it with the same arguments and reconstructs its own slab.
    Returns ``(volume, records)``: with ``gather="root"`` rank 0 gets the full
    ``Volume`` and other ranks ``None``; with ``gather="none"`` every rank gets its
    own slab as a device tensor.  ``on_record`` / ``snapshot_sink`` fire on rank
    0 only (snapshots gather the full volume every iteration -- tests only).
    ``transport`` is accepted for signature compatibility; the transport is the
    process group.  ``sino`` may also be the path of a saved sinogram: each rank
    then reads only its own rows (memory-mapped).  ``halo="peer"`` writes the halo
    planes straight into the neighbours' device memory (IPC-mapped inboxes,
    csrc/halo.cu) instead of sending them over the group.
    """
    src = _Rows(sino)
    if n_workers < 1:
        raise ValueError("need at least one worker")
    if n_workers > src.slices:
        raise ValueError("more workers than slices")
    if gather not in ("root", "none"):
        raise ValueError("gather must be 'root' or 'none'")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if n_workers != world and not (n_workers == 1 and world == 1):
        raise ValueError(f"n_workers={n_workers} must equal the process-group size {world} "
                         "(one process per GPU; launch with torchrun)")
    geom = ScanGeometry(angles=src.angles, detector_bins=src.detector_bins,
                        image_side=image_side)
    sampling = polar_sampling(geom)
    plan = NufftPlan(image_side, sampling, nufft_tolerance, oversampling)
    psf = build_psf(sampling, image_side, nufft_tolerance, oversampling)
    if f0 is not None and (f0.slices != src.slices or f0.side != image_side):
        raise ValueError("initial volume does not match the requested reconstruction")

    if n_workers == 1:
        L = cfg.lipschitz if cfg.lipschitz is not None else estimate_lipschitz(psf, params)
        cfg1 = SolverConfig(max_iters=cfg.max_iters, tol=cfg.tol, lipschitz=L,
                            restart=cfg.restart, log_every=cfg.log_every, nonneg=cfg.nonneg)
        ctx = fidelity_context(plan, psf, sino if isinstance(sino, Sinogram) else src.sinogram())
        x0 = f0 if f0 is not None else torch.zeros((src.slices, image_side, image_side),
                                                   device=_lib.device())
        vol, records = solve(ctx, params, cfg1, x0, on_record=on_record,
                             snapshot_sink=snapshot_sink)
        if isinstance(vol, torch.Tensor):
            if gather == "none":
                return vol, records
            vol = Volume._owned(_device.to_host64(vol))
        return vol, records

    rank = dist.get_rank(group)
    parts = partition(src.slices, n_workers)
    part = parts[rank]
    comm = SlabComm(part, group, halo=halo)
    try:
        L = cfg.lipschitz
        if L is None:
            L = comm.broadcast_scalar(estimate_lipschitz(psf, params) if rank == 0 else None)
        rows = src.rows(slice(part.begin, part.end))
        ctx = FidelityContext(psf=psf, rstar=back_project_stack(plan, rows),
                              g_norm_sq=float(np.sum(rows ** 2)))
        if f0 is None:
            x0 = torch.zeros((part.size, image_side, image_side), device=_lib.device())
        else:
            x0 = torch.from_numpy(np.ascontiguousarray(f0.data[part.begin:part.end],
                                                       dtype=np.float32)).to(_lib.device())
        stencil = stencil_3d() if src.slices > 1 else stencil_2d()
        sink = None
        if snapshot_sink is not None:
            def sink(k, slab):
                full = comm.gather(slab, parts)
                if rank == 0:
                    snapshot_sink(k, full.to("cpu", torch.float64).numpy())
        # the reference's record sink sees every record (runtime.py:654-659)
        slab, records = _iterate(ctx, params, cfg, x0, stencil, L, comm=comm,
                                 on_record=on_record if rank == 0 else None,
                                 device_snapshot=sink, x0_owned=True, log_filter=False)
        if gather == "none":
            return slab, records
        full = comm.gather(slab, parts)
        vol = Volume._owned(_device.to_host64(full)) if rank == 0 else None
        return vol, records
    except Exception as exc:  # noqa: BLE001 - any worker failure, divergence included,
        # surfaces as RuntimeError("worker i failed: ...") (runtime.py:684-690)
        raise RuntimeError(f"worker {rank} failed: {exc}") from exc


def distributed_solve_hierarchical(full_sino: Sinogram, hierarchy, params, cfg: SolverConfig,
                                   n_workers: int, *, use_fbp_init: bool = False,
                                   downsample_angles: bool = False,
                                   nufft_tolerance: float = 1e-6, oversampling: float = 2.0,
                                   on_record=None, gather: str = "root", group=None,
                                   halo: str = "nccl"):
    """Coarse-to-fine schedule over z-slabs (multires.py:198-242 x runtime.py:622-691).

    The reference never combines the two (cli.py:104-131); the north-star C4/C5
    runs need both.  Each level is re-partitioned (coarse and fine slabs do not
    nest), the level's sinogram rows of the slab are strided on the host, and the
    level solves with the slab loop of ``distributed_solve``.  Between levels the
    coarse estimate is all-gathered once (one-time per level) and every rank
    upsamples only its fine slab, so the Lanczos z-taps across slab boundaries
    see exactly the single-GPU inputs.  Returns ``(volume, per-level records)``
    as ``solve_hierarchical`` (volume on rank 0 with ``gather="root"``).
    """
    from .multires import _strided_indices, slab_source_range, upsample_slab
    from .radon import fbp_stack

    src = _Rows(full_sino)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if n_workers != world:
        raise ValueError(f"n_workers={n_workers} must equal the process-group size {world}")
    if world == 1:
        from .multires import solve_hierarchical

        full = full_sino if isinstance(full_sino, Sinogram) else src.sinogram()
        return solve_hierarchical(full, hierarchy, params, cfg, use_fbp_init=use_fbp_init,
                                  downsample_angles=downsample_angles,
                                  nufft_tolerance=nufft_tolerance, oversampling=oversampling,
                                  on_record=on_record)
    target = hierarchy.levels[-1]
    if src.detector_bins < target:
        raise ValueError("detector does not cover the target grid")
    rank = dist.get_rank(group)
    n_levels = len(hierarchy.levels)
    all_records, estimate, parts_prev = [], None, None
    for lvl, side in enumerate(hierarchy.levels):
        factor = 1 << (n_levels - 1 - lvl)
        bins = _strided_indices(src.detector_bins, factor) if factor > 1 else None
        zidx = (_strided_indices(src.slices, factor)
                if factor > 1 and src.slices > 1 else np.arange(src.slices))
        angles = src.angles
        keep = np.arange(0, angles.size, factor) if (downsample_angles and factor > 1) else None
        if keep is not None:
            angles = angles[keep]
        n_z = zidx.size
        if n_z < n_workers:
            raise ValueError(f"level {lvl} has {n_z} slices for {n_workers} workers")
        parts = partition(n_z, n_workers)
        part = parts[rank]
        rows = src.rows(zidx[part.begin:part.end])  # this rank's rows only
        if bins is not None:
            rows = rows[:, :, bins] / factor
        if keep is not None:
            rows = rows[:, keep, :]
        nd = rows.shape[2]
        geom = ScanGeometry(angles=angles, detector_bins=nd, image_side=side)
        sampling = polar_sampling(geom)
        plan = NufftPlan(side, sampling, nufft_tolerance, oversampling)
        psf = build_psf(sampling, side, nufft_tolerance, oversampling)
        comm = SlabComm(part, group, halo=halo)
        L = cfg.lipschitz
        if L is None:
            L = comm.broadcast_scalar(estimate_lipschitz(psf, params) if rank == 0 else None)
        ctx = FidelityContext(psf=psf, rstar=back_project_stack(plan, rows),
                              g_norm_sq=float(np.sum(rows ** 2)))
        if estimate is None:
            x0 = (fbp_stack(plan, rows) if use_fbp_init else
                  torch.zeros((part.size, side, side), device=_lib.device()))
        else:
            # only the coarse planes each fine slab's z-taps reach travel (p2p)
            ranges = [slab_source_range(parts_prev[-1].end, n_z, p.begin, p.end) for p in parts]
            coarse = SlabComm(parts_prev[rank], group).gather_range(estimate, parts_prev, ranges)
            estimate = None
            x0 = upsample_slab(coarse, side, n_z, part.begin, part.end, src_begin=ranges[rank][0],
                               n_src=parts_prev[-1].end)
        cfg_l = SolverConfig(max_iters=hierarchy.iters_per_level[lvl], tol=cfg.tol, lipschitz=L,
                             restart=cfg.restart, log_every=cfg.log_every, nonneg=cfg.nonneg)
        sink = ((lambda rec, _l=lvl: on_record(_l, rec))
                if (on_record is not None and rank == 0) else None)
        stencil = stencil_3d() if n_z > 1 else stencil_2d()
        estimate, records = _iterate(ctx, params, cfg_l, x0, stencil, L, comm=comm, on_record=sink,
                                     x0_owned=True, log_filter=False)
        all_records.append(records)
        parts_prev = parts
    if gather == "none":
        return estimate, all_records
    full = SlabComm(parts_prev[rank], group).gather(estimate, parts_prev)
    vol = Volume._owned(_device.to_host64(full)) if rank == 0 else None
    return vol, all_records
