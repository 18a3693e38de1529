"""Shared fixtures.  Tests marked ``gpu`` need a B200 (they call libdhgp.so);
everything else runs on the CPU (oracle vs golden fixtures, host logic,
library symbol table, multi-process gloo)."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"

# The worked example H1 of the reference tests (conftest.py:12 there).
H1_TEXT = "3 4\n1 1 2 0 1 2\n2 1 1 1 2\n1 1 1 3 0\n"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (libdhgp.so on sm_100a)")


@pytest.fixture
def h1():
    import paper_2604_14411_b200 as dp

    return dp.parse_dhg_host(H1_TEXT)


def arrays_of(g):
    return (g.num_nodes, g.edge_weight, g.edge_src.offsets, g.edge_src.data, g.edge_dst.offsets, g.edge_dst.data)


def make_instance(num_nodes, num_edges, max_pins, seed, omega, delta_slack=0):
    """Reference conftest.make_instance: generated graph + feasible limits."""
    import paper_2604_14411_b200 as dp
    from paper_2604_14411_b200 import workloads as W

    n, w, so, sd, do, dd = W.random_dhg(num_nodes, num_edges, max_pins, seed=seed)
    g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
    indeg = int(np.bincount(dd, minlength=n).max()) if len(dd) else 0
    return g, dp.Constraints(omega, max(indeg, 1) + delta_slack)


def load_npz(name):
    return np.load(GOLDEN / name, allow_pickle=False)
