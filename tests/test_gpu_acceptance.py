"""Quality acceptance on GPU results: the reference's acceptance criteria 7
and 8 (pkg/tests/test_acceptance.py:249-300), restated.  Bit-exact parity with
the reference is proven elsewhere; these check that the GPU partitioner's
output also clears the reference's own quality bars."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import make_instance

pytestmark = pytest.mark.gpu


def _optimum(g, c):
    """Smallest connectivity over every valid set partition (restricted-growth
    enumeration; test-only brute force for n <= 8, cf. oracles.py:49-100)."""
    n = g.num_nodes
    inb = [set(g.node_in.segment(v).tolist()) for v in range(n)]
    sz = [int(s) for s in g.node_size]
    pins = [g.edge_pins.segment(e).tolist() for e in range(g.num_edges)]
    w = [float(x) for x in g.edge_weight]
    assign = [0] * n
    psize = [0] * (n + 1)
    pin_sets = [set() for _ in range(n + 1)]
    best = [float("inf")]

    def rec(i, used):
        if i == n:
            conn = sum(we * (len({assign[v] for v in e}) - 1) for we, e in zip(w, pins) if e)
            best[0] = min(best[0], conn)
            return
        for p in range(used + 1):
            if psize[p] + sz[i] > c.max_size or len(pin_sets[p] | inb[i]) > c.max_inbound:
                continue
            saved = pin_sets[p]
            assign[i], psize[p], pin_sets[p] = p, psize[p] + sz[i], saved | inb[i]
            rec(i + 1, max(used, p + 1))
            psize[p] -= sz[i]
            pin_sets[p] = saved

    rec(0, 0)
    return best[0]


def test_quality_vs_baselines():
    import paper_2604_14411_b200 as d

    rs = np.random.RandomState(4242)
    ours, onep, over = [], [], []
    for i in range(50):
        n = int(rs.randint(40, 161))
        omega = int(rs.choice([4, 8, 16]))
        g, c = make_instance(n, int(1.5 * n), 5, seed=40_000 + i, omega=omega, delta_slack=omega)
        part, _ = d.partition(g, d.Config(c))
        ours.append(d.connectivity(g, part))
        onep.append(d.connectivity(g, d.one_pass(g, c)))
        over.append(d.connectivity(g, d.overlap_greedy(g, c)))
    assert np.mean(ours) / np.mean(onep) <= 0.9
    assert np.mean(ours) / np.mean(over) <= 1.0


def test_brute_force_sanity():
    import paper_2604_14411_b200 as d

    rs = np.random.RandomState(77)
    beat_or_tie = 0
    for i in range(30):
        n = int(rs.randint(4, 9))
        omega = int(rs.choice([2, 3, 4]))
        g, c = make_instance(n, n + int(rs.randint(2, 6)), min(4, n), seed=50_000 + i, omega=omega, delta_slack=1)
        part, _ = d.partition(g, d.Config(c))
        conn = d.connectivity(g, part)
        assert d.check_validity(g, part, c) == []
        assert conn >= _optimum(g, c)
        beat_or_tie += conn <= d.connectivity(g, d.one_pass(g, c))
    assert beat_or_tie >= 24


def test_batch_size_invariance():
    """Criterion 6 (test_acceptance.py:222-246) at the partition level: the
    histogram batch changes no output (fill_histograms is batch-invariant)."""
    import paper_2604_14411_b200 as d

    rs = np.random.RandomState(661)
    for i in range(20):
        n = int(rs.randint(30, 301))
        omega = int(rs.choice([4, 8, 16]))
        g, c = make_instance(n, int(1.5 * n), 5, seed=30_000 + i, omega=omega, delta_slack=omega)
        ref, rst = d.partition(g, d.Config(c, batch_size=1))
        for b in (7, 32):
            got, st = d.partition(g, d.Config(c, batch_size=b))
            assert ref.assign.tobytes() == got.assign.tobytes() and rst.to_dict() == st.to_dict()


def test_pin_scaling():
    """Criterion 10 (test_acceptance.py:334-360): partition time grows at most
    2.5x per doubling of the pins.

    At these sizes a run is ~4 ms of launch latency (the same 784 launches at
    every size), so host scheduling bursts on the box (10-90 ms stalls seen
    on a freshly acquired machine) swamp a median of five.  The sizes are
    timed round-robin and each size's statistic is its fastest of nine runs:
    the run's own cost, without the machine's noise.
    """
    import time

    import paper_2604_14411_b200 as d
    from paper_2604_14411_b200 import workloads as W

    cases = []
    for nodes, edges in ((2000, 2500), (4000, 5000), (8000, 10000)):
        n, w, so, sd, do, dd = W.random_dhg(nodes, edges, 6, seed=2)
        g = d.Hypergraph._from_csr(n, w, d.CsrSets(so, sd), d.CsrSets(do, dd))
        cases.append((g, d.Config(d.Constraints(16, max(int(g.node_in.lengths().max()), 24)))))
        d.partition(*cases[-1])
    best = [float("inf")] * len(cases)
    for _ in range(9):
        for i, (g, cfg) in enumerate(cases):
            t0 = time.perf_counter()
            d.partition(g, cfg)
            best[i] = min(best[i], time.perf_counter() - t0)
    assert best[1] / best[0] <= 2.5 and best[2] / best[1] <= 2.5, best
