"""Comparison baselines on the GPU: the reference's one-pass filler and
incidence-overlap greedy (baselines.py:16-91), bit-identical.

Both are sequential greedy procedures by definition; ``libdhgp.so`` runs each
as one persistent kernel (csrc/baselines.cu), with the parallelism inside a
decision.  They are the quality reference points of the paper's comparison
 at sizes the reference's Python loops cannot reach.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .hgraph import Constraints, Hypergraph, Partitioning

__all__ = ["one_pass", "overlap_greedy"]


def _run(g: Hypergraph, c: Constraints, method: int) -> Partitioning:
    L = _lib.load()
    gg, keep = g._c_graph()
    assign = np.zeros(max(g.num_nodes, 1), dtype=np.int32)
    nparts = C.c_int32(0)
    rc = L.dhgp_baseline(C.byref(gg), C.c_int64(c.max_size), C.c_int64(c.max_inbound), C.c_int32(method),
                         C.c_int32(_lib.device()), _lib.ptr(assign), C.byref(nparts))
    del keep
    _lib.raise_for(rc)
    return Partitioning(assign[:g.num_nodes].copy(), int(nparts.value))


def one_pass(g: Hypergraph, c: Constraints) -> Partitioning:
    """Nodes in id order fill one open partition; a node that would exceed
    max_size or the distinct-inbound bound opens the next (baselines.py:16-40)."""
    return _run(g, c, 0)


def overlap_greedy(g: Hypergraph, c: Constraints) -> Partitioning:
    """Seed the lowest unassigned id, then repeatedly add the free node with
    the largest incident-edge overlap with the partition (ties to the smaller
    id) while the overlap is positive and both bounds hold
    (baselines.py:43-91)."""
    return _run(g, c, 1)
