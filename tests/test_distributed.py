"""Node-range sharding.

CPU tier: the shard rule (Python mirror vs the library's own C rule, through
the C-ABI), and the host allgather over a real world_size-2/3 gloo group.
GPU tier: several processes on cuda:0 running the sharded partition over the
host transport (every phase sharded) must reproduce the single-GPU result bit
for bit; the NCCL transport is initialised and used at world size 1.
"""
from __future__ import annotations

import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ---------------------------------------------------------------------------
# CPU tier
# ---------------------------------------------------------------------------
def test_shard_rule_matches_library_and_covers_every_unit():
    from paper_2604_14411_b200 import _lib
    from paper_2604_14411_b200.distributed import shard_range

    L = _lib.load(require_device=False)
    lo, hi, ch = C.c_int64(), C.c_int64(), C.c_int64()
    for world in (1, 2, 3, 4, 7, 8):
        for n in (0, 1, 2, 5, 17, 1000, 65535, 65536, 100003):
            for mu in (0, 16, 65536):
                covered = []
                for rank in range(world):
                    on = L.dhgp_shard_range(world, rank, C.c_int64(mu), C.c_int64(n), C.byref(lo), C.byref(hi),
                                            C.byref(ch))
                    py = shard_range(n, world, rank, mu)
                    assert (bool(on), lo.value, hi.value, ch.value) == py
                    if on:
                        assert ch.value * world >= n and lo.value == min(n, rank * ch.value)
                        covered.extend(range(lo.value, hi.value))
                    else:
                        assert (lo.value, hi.value) == (0, n)
                if covered:
                    assert covered == list(range(n))


def _gather_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        from paper_2604_14411_b200.distributed import host_allgather_fn

        fn = host_allgather_fn()
        nbytes = 13
        buf = (C.c_uint8 * (nbytes * world))()
        arr = np.ctypeslib.as_array(buf)
        arr[:] = 255
        arr[rank * nbytes:(rank + 1) * nbytes] = np.arange(nbytes, dtype=np.uint8) + 10 * rank
        rc = fn(None, C.addressof(buf), nbytes)
        want = np.concatenate([np.arange(nbytes, dtype=np.uint8) + 10 * r for r in range(world)])
        q.put((rank, rc, bool(np.array_equal(arr, want))))
    except BaseException as ex:  # surfaced in the parent
        q.put((rank, -1, repr(ex)))


@pytest.mark.parametrize("world", [2, 3])
def test_host_allgather_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert [r[1:] for r in res] == [(0, True)] * world, res


def _comm_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        from paper_2604_14411_b200.distributed import Communicator

        cm = Communicator.host()
        cm.set_min_units(0)
        st = cm.stats()
        cm.close()
        q.put((rank, st["allgathers"], cm.world, cm.rank))
    except BaseException as ex:
        q.put((rank, -1, repr(ex), None))


def test_host_communicator_lifecycle_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_comm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert res == [(0, 0, 2, 0), (1, 0, 2, 1)], res


# ---------------------------------------------------------------------------
# GPU tier
# ---------------------------------------------------------------------------
def _instances():
    from conftest import make_instance

    from paper_2604_14411_b200 import workloads as W
    import paper_2604_14411_b200 as dp

    out = []
    for t, (n, om) in enumerate(((300, 16), (700, 32), (1200, 64))):
        g, c = make_instance(n, 2 * n, 6, seed=4400 + t, omega=om, delta_slack=20)
        out.append((g, c.max_size, c.max_inbound))
    n, w, so, sd, do, dd = W.layered_snn(6, 300, fanout=32, window=128, seed=2)
    out.append((dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd)), 256, 4096))
    return out


def _large_instances():
    """Above the default min_units (65,536 nodes / h-edges): the sharded
    phases run with the library's default threshold."""
    import paper_2604_14411_b200 as dp
    from paper_2604_14411_b200 import workloads as W

    n, w, so, sd, do, dd = W.layered_snn(70, 1000, seed=5)
    return [(dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd)), 1024, 4096)]


def _sharded_worker(rank, world, port, q, default_min_units=False):
    try:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parent))
        _init(rank, world, port)
        import paper_2604_14411_b200 as dp
        from paper_2604_14411_b200 import distributed as dd

        cm = dd.Communicator.host()
        if not default_min_units:
            cm.set_min_units(0)  # shard every level and every round
        out = []
        for g, om, de in (_large_instances() if default_min_units else _instances()):
            part, st = dd.partition(g, dp.Config(dp.Constraints(om, de), max_levels=1 << 20), cm)
            out.append((part.assign.tobytes(), part.num_parts, st.levels, st.connectivity_trace))
        q.put((rank, out, cm.stats()["allgathers"]))
        cm.close()
    except BaseException as ex:
        import traceback

        q.put((rank, None, traceback.format_exc() + repr(ex)))


@pytest.mark.gpu
@pytest.mark.parametrize("world,default_min_units", [(2, False), (3, False), (2, True)])
def test_sharded_partition_is_bit_identical(world, default_min_units):
    """Node-range sharding (full and incremental scoring, proposals, the
    in-sequence gain / inbound terms by h-edge range) over world 2/3 ranks on
    one GPU with the host (gloo) allgather: every rank's result equals the
    single-GPU one.  min_units 0 shards every level and round; the default
    threshold (65,536) shards the 70k-node instance's large phases."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import paper_2604_14411_b200 as dp

    ref = []
    for g, om, de in (_large_instances() if default_min_units else _instances()):
        part, st = dp.partition(g, dp.Config(dp.Constraints(om, de), max_levels=1 << 20))
        ref.append((part.assign.tobytes(), part.num_parts, st.levels, st.connectivity_trace))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_sharded_worker, args=(r, world, port, q, default_min_units)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda x: x[0])
    for p in ps:
        p.join(timeout=120)
    for rank, out, calls in res:
        assert out is not None, calls
        assert calls > 0, "no exchange happened"
        for i, (a, b) in enumerate(zip(out, ref)):
            assert a == b, f"rank {rank} instance {i} differs from the single-GPU result"


@pytest.mark.gpu
def test_nccl_communicator_world1():
    import torch.distributed as dist

    import paper_2604_14411_b200 as dp
    from paper_2604_14411_b200 import distributed as dd

    port = _free_port()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["DHGP_COMM_EXERCISE"] = "1"  # issue the in-place ncclAllGather even at world size 1
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        cm = dd.Communicator.nccl()
        cm.set_min_units(0)
        for g, om, de in _instances():
            cfg = dp.Config(dp.Constraints(om, de), max_levels=1 << 20)
            a, sa = dd.partition(g, cfg, cm)
            b, sb = dp.partition(g, cfg)
            assert np.array_equal(a.assign, b.assign) and sa.connectivity_trace == sb.connectivity_trace
        assert cm.stats()["allgathers"] > 0
        cm.close()
    finally:
        os.environ.pop("DHGP_COMM_EXERCISE", None)
        dist.destroy_process_group()
