"""Multi-GPU partitioning by node-range sharding.

One process per GPU.  Each rank holds a replica of the hypergraph and of every
coarsening level; candidate scoring (coarsen.py:93-132) and move proposals
(refine.py:82-116) — the per-node phases whose work is the sum of the
neighbourhood sizes — are computed for the rank's node range and completed
by an in-place allgather inside ``libdhgp.so``; the rest of the pipeline
(contraction, matching, the O(sum |e|) sequence gains, the event pipeline)
runs replicated.  The exchanged
values are exact (int32 ids, int64 gains, f64 scores) and every tie-break is
the reference's global total order, so every rank returns the same result as
the single-GPU :func:`partition` — bit for bit, at any world size.

Two transports:

* :meth:`Communicator.nccl` — ``ncclAllGather`` on the library's CUDA stream
  over NVLink / NVSwitch (the NCCL unique id is broadcast through
  ``torch.distributed``);
* :meth:`Communicator.host` — the allgather runs on the host through
  ``torch.distributed`` (any backend, e.g. gloo); used to exercise the sharded
  path with several processes on one GPU, and on hosts without NCCL.

The reference has no multi-process mode; this module is the §8(e) extension
of its ``partition`` entry point (driver.py:76-163).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

__all__ = ["Communicator", "partition", "shard_range", "host_allgather_fn"]

ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64)

DEFAULT_MIN_UNITS = 1 << 16


def shard_range(n: int, world: int, rank: int, min_units: int = DEFAULT_MIN_UNITS) -> tuple[bool, int, int, int]:
    """(sharded, lo, hi, chunk) of ``rank`` over ``n`` units — the rule
    libdhgp applies to every sharded phase (csrc/comm.cu ``shard_of``)."""
    if world <= 1 or n <= 0 or n < min_units:
        return False, 0, n, n
    chunk = -(-n // world)
    lo = min(n, rank * chunk)
    return True, lo, min(n, lo + chunk), chunk


def host_allgather_fn(group=None):
    """A ``dhgp_allgather_fn`` body over ``torch.distributed`` (any backend):
    ``buf`` holds world * nbytes bytes, this rank's part at rank * nbytes;
    returns 0 after every part is filled in."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)

    def fn(_user, buf, nbytes):
        try:
            arr = np.ctypeslib.as_array((C.c_uint8 * (nbytes * world)).from_address(buf))
            mine = torch.from_numpy(arr[rank * nbytes:(rank + 1) * nbytes].copy())
            parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, mine, group=group)
            for r in range(world):
                arr[r * nbytes:(r + 1) * nbytes] = parts[r].numpy()
            return 0
        except BaseException:  # reported to the library as a failed exchange
            return 1

    return fn


class Communicator:
    """A libdhgp communicator (``dhgp_comm``) for this process's rank."""

    def __init__(self, handle, world: int, rank: int, keep=None):
        self._h = handle
        self.world = world
        self.rank = rank
        self._keep = keep

    @classmethod
    def nccl(cls, group=None, device: int | None = None) -> "Communicator":
        """NCCL transport; ``torch.distributed`` must be initialised (any
        backend) and carries the unique id from rank 0."""
        import torch.distributed as dist

        L = _lib.load()
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _lib.raise_for(L.dhgp_comm_nccl_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        dev = _lib.device() if device is None else int(device)
        _lib.raise_for(L.dhgp_comm_init_nccl(world, rank, uid, dev, C.byref(h)))
        return cls(h, world, rank)

    @classmethod
    def host(cls, group=None) -> "Communicator":
        """Host transport over ``torch.distributed`` (e.g. gloo)."""
        import torch.distributed as dist

        L = _lib.load(require_device=False)
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        cb = ALLGATHER(host_allgather_fn(group))
        h = C.c_void_p()
        _lib.raise_for(L.dhgp_comm_init_host(world, rank, cb, None, C.byref(h)))
        return cls(h, world, rank, keep=cb)

    def set_min_units(self, n: int) -> None:
        """Phases over fewer than ``n`` nodes / moves run replicated."""
        _lib.raise_for(_lib.load(require_device=False).dhgp_comm_set_min_units(self._h, C.c_int64(int(n))))

    def stats(self) -> dict:
        calls, nbytes = C.c_int64(0), C.c_double(0)
        _lib.load(require_device=False).dhgp_comm_stats(self._h, C.byref(calls), C.byref(nbytes))
        return {"allgathers": int(calls.value), "bytes_received": float(nbytes.value)}

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if self._h:
            _lib.load(require_device=False).dhgp_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition(g, cfg, comm: Communicator, timings: bool = False):
    """Sharded :func:`paper_2604_14411_b200.partition`: every rank calls it
    with the same graph and config and gets the same (Partitioning, RunStats)."""
    from .driver import _make_config, _stats_from
    from .hgraph import ID, Partitioning

    L = _lib.load()
    gg, keep = g._c_graph()
    cc = _make_config(cfg)
    assign = np.zeros(max(g.num_nodes, 1), dtype=ID)
    nparts = C.c_int32(0)
    st = _lib.DhgpStats()
    rc = L.dhgp_partition_sharded(C.byref(gg), C.byref(cc), comm.handle, _lib.ptr(assign), C.byref(nparts),
                                  C.byref(st))
    del keep
    _lib.raise_for(rc)
    stats = _stats_from(L, st, timings)
    return Partitioning(assign[: g.num_nodes].copy(), int(nparts.value)), stats
