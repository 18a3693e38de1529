"""The drop-in entry point: ``partition(g, cfg, observer=None, timings=False)``.

Same signature, return types, exceptions and observer payloads as
dhgpart.driver.partition (driver.py:76-163).  The whole multi-level loop —
incidence, coarsening levels, initial partitioning, refinement rounds,
compaction and the validity check — runs inside libdhgp.so on the GPU
(``dhgp_partition``); this module only marshals arguments and results.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .coarsen import ClusterMap, PairingForest
from .hgraph import ID, Constraints, CsrSets, Hypergraph, Partitioning
from .refine import MoveSet, PrefixSelection

__all__ = ["Config", "RunStats", "partition"]


@dataclass(frozen=True)
class Config:
    """Partitioner knobs (driver.py:31-52).  ``seed`` is accepted and unused
    (the pipeline is deterministic); ``batch_size`` is validated but cannot
    change the result (histogram batching is a memory-traffic knob in the
    reference; here the histogram never leaves shared memory)."""

    constraints: Constraints
    max_rounds: int = 8
    batch_size: int = 32
    seed: int = 0
    max_levels: int = 64

    def __post_init__(self):
        for name in ("max_rounds", "batch_size", "max_levels"):
            v = getattr(self, name)
            if v < 1:
                raise ValueError(f"{name} must be >= 1, got {v}")


@dataclass
class RunStats:
    """Per-level sizes (finest first), connectivity trace per refinement
    stage (coarsest first), optional phase wall times, final part count."""

    levels: list[dict] = field(default_factory=list)
    connectivity_trace: list[list[float]] = field(default_factory=list)
    phase_ms: dict = field(default_factory=dict)
    num_partitions: int = 0

    def to_dict(self) -> dict:
        return {
            "levels": self.levels,
            "connectivity_trace": self.connectivity_trace,
            "phase_ms": self.phase_ms,
            "num_partitions": self.num_partitions,
        }


def _make_config(cfg: Config) -> _lib.DhgpConfig:
    c = cfg.constraints
    return _lib.DhgpConfig(int(c.max_size), int(c.max_inbound), int(cfg.max_rounds), int(cfg.batch_size),
                           int(cfg.max_levels), _lib.device())


class _ObserverBridge:
    """Turns libdhgp observer events into the reference's payload objects."""

    def __init__(self, g: Hypergraph, observer):
        self.observer = observer
        self.levels = [g]
        self.error = None

    def __call__(self, evp, _user):
        if self.error is not None:
            return
        try:
            ev = evp.contents
            if ev.kind == 1:
                n, nc, E = ev.num_nodes, ev.num_coarse, ev.num_edges
                so = _lib.take(ev.c_src_off, E + 1, np.int64)
                do = _lib.take(ev.c_dst_off, E + 1, np.int64)
                fine = self.levels[ev.level]
                coarse = Hypergraph._from_csr(
                    nc, fine.edge_weight,
                    CsrSets(so, _lib.take(ev.c_src_dat, int(so[-1]), ID)),
                    CsrSets(do, _lib.take(ev.c_dst_dat, int(do[-1]), ID)),
                    node_size=_lib.take(ev.c_node_size, nc, ID),
                )
                self.levels.append(coarse)
                forest = PairingForest(pair=_lib.take(ev.pair, n, np.int32), score=_lib.take(ev.score, n, np.float64),
                                       match=_lib.take(ev.match, n, np.int32))
                cmap = ClusterMap(gamma=_lib.take(ev.gamma, n, ID), num_coarse=nc)
                self.observer("level", {"index": ev.level, "fine": fine, "coarse": coarse, "forest": forest,
                                        "cmap": cmap})
            else:
                m = ev.num_moves
                moves = MoveSet(
                    node=_lib.take(ev.mv_node, m, ID), from_part=_lib.take(ev.mv_from, m, ID),
                    to_part=_lib.take(ev.mv_to, m, ID), gain_iso=_lib.take(ev.mv_gain_iso, m, np.float64),
                    gain_seq=_lib.take(ev.mv_gain_seq, m, np.float64),
                )
                sel = PrefixSelection(int(ev.k), float(ev.total_gain), _lib.take(ev.active, m + 1, np.int64))
                self.observer("round", {
                    "level": ev.level, "round": ev.round, "graph": self.levels[ev.level],
                    "num_parts": ev.num_parts, "assign": _lib.take(ev.assign, ev.num_nodes, ID),
                    "moves": moves, "selection": sel,
                })
        except BaseException as ex:  # re-raised after the C call returns
            self.error = ex


def partition(g: Hypergraph, cfg: Config, observer=None, timings: bool = False) -> tuple[Partitioning, RunStats]:
    """Partition ``g`` under ``cfg.constraints``, minimising connectivity.

    Raises InfeasibleError when no valid partitioning exists, DhgError when
    coarsening needs more than ``cfg.max_levels`` levels, and
    MatchingInvariantError on a broken pairing forest — as the reference.
    """
    L = _lib.load()
    gg, keep = g._c_graph()
    cc = _make_config(cfg)
    assign = np.zeros(max(g.num_nodes, 1), dtype=ID)
    nparts = C.c_int32(0)
    st = _lib.DhgpStats()
    bridge = _ObserverBridge(g, observer) if observer is not None else None
    cb = _lib.OBSERVER(bridge) if bridge is not None else _lib.OBSERVER()
    rc = L.dhgp_partition(C.byref(gg), C.byref(cc), _lib.ptr(assign), C.byref(nparts), C.byref(st), cb, None)
    del keep
    if bridge is not None and bridge.error is not None:
        if rc == _lib.OK:
            L.dhgp_stats_free(C.byref(st))
        raise bridge.error
    _lib.raise_for(rc)
    stats = _stats_from(L, st, timings)
    return Partitioning(assign[: g.num_nodes].copy(), int(nparts.value)), stats


def _stats_from(L, st, timings: bool) -> RunStats:
    """RunStats from a filled dhgp_stats (frees the library's buffers)."""
    try:
        nl = st.num_levels
        tro = _lib.take(st.trace_off, nl + 1, np.int64)
        trv = _lib.take(st.trace_val, int(tro[-1]) if nl >= 0 else 0, np.float64)
        stats = RunStats(
            levels=[{"nodes": int(st.level_nodes[i]), "edges": int(st.level_edges[i]),
                     "pins": int(st.level_pins[i])} for i in range(nl)],
            connectivity_trace=[[float(x) for x in trv[tro[i]:tro[i + 1]]] for i in range(nl)],
            num_partitions=int(st.num_partitions),
        )
        if timings:
            stats.phase_ms = {"coarsen": float(st.phase_ms[0]), "refine": float(st.phase_ms[1]),
                              "total": float(st.phase_ms[2])}
        stats._gpu_launches = int(st.gpu_launches)  # not part of to_dict()
    finally:
        L.dhgp_stats_free(C.byref(st))
    return stats
