"""Coarsening payload types and the neighbour-set API (coarsen.py:44-85).

The coarsening itself (scoring, selection, matching, contraction) runs on
the GPU inside ``dhgp_partition``; these classes carry its per-level results
to the observer exactly as the reference's do.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .hgraph import ID, OFFSET, CsrSets, Hypergraph

__all__ = ["PairingForest", "ClusterMap", "materialize_neighbors"]


@dataclass(frozen=True)
class PairingForest:
    """Per-node candidate ``pair`` (-1 = none), its histogram ``score`` and
    the final ``match`` involution (``match[n] == n`` for singletons)."""

    pair: np.ndarray
    score: np.ndarray
    match: np.ndarray | None = None

    def matched_pairs(self) -> int:
        if self.match is None:
            return 0
        return int(np.count_nonzero(self.match != np.arange(len(self.match)))) // 2


@dataclass(frozen=True)
class ClusterMap:
    """Fine node -> coarse node map of one contraction; coarse ids ascend
    with each cluster's minimum fine id."""

    gamma: np.ndarray
    num_coarse: int

    def members(self) -> CsrSets:
        """Coarse node -> sorted fine member ids."""
        order = np.argsort(self.gamma, kind="stable")
        counts = np.bincount(self.gamma, minlength=self.num_coarse)
        off = np.zeros(self.num_coarse + 1, dtype=OFFSET)
        np.cumsum(counts, out=off[1:])
        return CsrSets(off, order.astype(ID))


def materialize_neighbors(g: Hypergraph) -> CsrSets:
    """Sorted unique neighbour set per node (coarsen.py:78-85), on the GPU."""
    L = _lib.load()
    gg, keep = g._c_graph()
    off = np.zeros(g.num_nodes + 1, dtype=OFFSET)
    dat = C.POINTER(C.c_int32)()
    nnz = C.c_int64(0)
    rc = L.dhgp_neighbors(C.byref(gg), C.c_int32(_lib.device()), _lib.ptr(off), C.byref(dat), C.byref(nnz))
    del keep
    _lib.raise_for(rc)
    try:
        data = _lib.take(dat, nnz.value, ID)
    finally:
        L.dhgp_free(dat)
    return CsrSets(off, data)
