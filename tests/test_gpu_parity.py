"""GPU parity: libdhgp.so (through the public API and the C-ABI seams) against
the reference's golden fixtures and the CPU oracle.  Bit-exact equality for
every integer and f64 output (weights are integral)."""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import H1_TEXT, arrays_of, load_npz, make_instance
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def dp():
    import paper_2604_14411_b200 as m

    return m


def graph(arr):
    d = dp()
    n, w, so, sd, do, dd = arr
    return d.Hypergraph._from_csr(int(n), w, d.CsrSets(so, sd), d.CsrSets(do, dd))


def run_gpu(g, omega, delta, record=False, **kw):
    d = dp()
    ev = []

    def obs(kind, p):
        ev.append((kind, p))

    part, st = d.partition(g, d.Config(d.Constraints(omega, delta), **kw), observer=obs if record else None)
    return part, st, ev


def assert_same_as_oracle(g, omega, delta, max_levels=1 << 20, **kw):
    part, st, _ = run_gpu(g, omega, delta, max_levels=max_levels, **kw)
    a, k, ost, _ = orc.partition(*arrays_of(g), g.node_size, max_size=omega, max_inbound=delta,
                                 max_levels=max_levels, **kw)
    assert np.array_equal(part.assign, a)
    assert part.num_parts == k == st.num_partitions
    assert st.levels == ost["levels"]
    assert st.connectivity_trace == ost["connectivity_trace"]
    return part, st


# ---------------------------------------------------------------------------
# golden fixtures from the reference
# ---------------------------------------------------------------------------
def test_partition_small_golden_with_observer_payloads():
    z = load_npz("partition_small.npz")
    for t in z["cases"]:
        check_golden_case(z, t)


def check_golden_case(z, t):
    """partition() of fixture case t against the reference's outputs and
    every per-level / per-round observer payload it recorded."""
    if True:
        p = f"c{t}_"
        g = graph([z[f"{p}in_{k}"] for k in ("n", "w", "so", "sd", "do", "dd")])
        part, st, ev = run_gpu(g, int(z[p + "omega"]), int(z[p + "delta"]), record=True, max_levels=1 << 20)
        ref = json.loads(bytes(z[p + "stats"]).decode())
        assert np.array_equal(part.assign, z[p + "assign"]), t
        assert part.num_parts == int(z[p + "num_parts"])
        assert st.levels == ref["levels"] and st.connectivity_trace == ref["trace"]
        lev = [e for k, e in ev if k == "level"]
        rnd = [e for k, e in ev if k == "round"]
        assert len(lev) == int(z[p + "nlev_ev"]) and len(rnd) == int(z[p + "nround_ev"])
        for i, e in enumerate(lev):
            f, cm, co = e["forest"], e["cmap"], e["coarse"]
            assert e["index"] == i and co.num_nodes == cm.num_coarse
            for got, fk in ((f.pair, "pair"), (f.score, "score"), (f.match, "match"), (cm.gamma, "gamma"),
                            (co.edge_src.offsets, "so"), (co.edge_src.data, "sd"), (co.edge_dst.offsets, "do"),
                            (co.edge_dst.data, "dd"), (co.node_size, "size")):
                assert np.array_equal(got, z[f"{p}L{i}_{fk}"]), (t, i, fk)
        for i, e in enumerate(rnd):
            m, s = e["moves"], e["selection"]
            assert e["level"] == int(z[f"{p}R{i}_level"]) and e["round"] == int(z[f"{p}R{i}_round"])
            for got, fk in ((e["assign"], "assign"), (m.node, "node"), (m.from_part, "from"), (m.to_part, "to"),
                            (m.gain_iso, "giso"), (m.gain_seq, "gseq"), (s.active, "active")):
                assert np.array_equal(got, z[f"{p}R{i}_{fk}"]), (t, i, fk)
            assert s.k == int(z[f"{p}R{i}_k"]) and s.total_gain == float(z[f"{p}R{i}_total"])


@pytest.mark.parametrize("name,gen,omega,delta", [
    ("c1.npz", ("random_dhg", dict(num_nodes=10_000, num_edges=20_000, max_pins=8, seed=0)), 256, 1024),
    ("snn.npz", ("layered_snn", dict(layers=3, width=300)), 64, 4096),
])
def test_full_instances_golden(name, gen, omega, delta):
    from paper_2604_14411_b200 import workloads as W

    z = load_npz(name)
    g = graph(getattr(W, gen[0])(**gen[1]))
    part, st, _ = run_gpu(g, omega, delta, max_levels=1 << 20)
    ref = json.loads(bytes(z["stats"]).decode())
    assert np.array_equal(part.assign, z["assign"])
    assert part.num_parts == int(z["num_parts"])
    assert st.levels == ref["levels"] and st.connectivity_trace == ref["trace"]


def test_kernel_seams_match_reference():
    from paper_2604_14411_b200 import kernels as K

    z = load_npz("kernels.npz")
    d = dp()
    for t in range(int(z["count"])):
        p = f"k{t}_"
        g = graph([z[f"{p}in_{k}"] for k in ("n", "w", "so", "sd", "do", "dd")])
        w = g.edge_weight
        assert np.array_equal(g.edge_pins.data, z[p + "pin_dat"]) and np.array_equal(g.node_inc.data, z[p + "inc_dat"])
        assert np.array_equal(g.node_in.offsets, z[p + "in_off"]) and np.array_equal(g.node_in.data, z[p + "in_dat"])
        assert np.array_equal(g.node_out.data, z[p + "out_dat"])
        nb = d.materialize_neighbors(g)
        assert np.array_equal(nb.offsets, z[p + "nb_off"]) and np.array_equal(nb.data, z[p + "nb_dat"])
        for batch in (1, 7, 32):
            hist = K.fill_histograms(g.node_inc.offsets, g.node_inc.data, g.edge_pins.offsets, g.edge_pins.data,
                                     w, nb.offsets, nb.data, batch)
            assert np.array_equal(hist, z[p + "hist"])
        pair, score = K.select_first_valid(z[p + "order"], nb.offsets, nb.data, hist, g.node_size,
                                           g.node_in.offsets, g.node_in.data, int(z[p + "omega"]),
                                           int(z[p + "delta"]))
        assert np.array_equal(pair, z[p + "pair"]) and np.array_equal(score, z[p + "score"])
        assert np.array_equal(K.resolve_matching(pair, score), z[p + "match"])
        assign = z[p + "assign"]
        assert K.connectivity_value(g.edge_pins.offsets, g.edge_pins.data, w, assign) == float(z[p + "conn"])
        kk = int(z[p + "K"])
        pins, pins_in = K.compute_pins(g.edge_pins.offsets, g.edge_pins.data, g.edge_dst.offsets, g.edge_dst.data,
                                       assign, kk)
        assert np.array_equal(pins, z[p + "pins"]) and np.array_equal(pins_in, z[p + "pins_in"])
        assert np.array_equal(d.partition_sizes(g, assign, kk), z[p + "psz"])
        assert np.array_equal(d.distinct_inbound_sizes(g, assign, kk), z[p + "pinb"])
        tgt, gain = K.propose_moves(g.node_inc.offsets, g.node_inc.data, g.edge_pins.offsets, g.edge_pins.data, w,
                                    pins, assign, z[p + "psz"], g.node_size, int(z[p + "omega"]))
        assert np.array_equal(tgt, z[p + "target"]) and np.array_equal(gain, z[p + "gain"])
        node = z[p + "node"]
        gseq = K.sequence_gains(g.node_inc.offsets, g.node_inc.data, g.edge_pins.offsets, g.edge_pins.data, w, pins,
                                node, assign[node], tgt[node], gain[node], z[p + "pos"])
        assert np.array_equal(gseq, z[p + "gseq"])
        k, tg, active = K.build_events_and_select(g.num_nodes, g.node_in.offsets, g.node_in.data, g.node_size, node,
                                                  assign[node], tgt[node], gseq, pins_in, z[p + "psz"],
                                                  z[p + "pinb"], int(z[p + "omega"]), int(z[p + "delta"]))
        assert k == int(z[p + "sel_k"]) and tg == float(z[p + "sel_total"])
        assert np.array_equal(active, z[p + "sel_active"])


# ---------------------------------------------------------------------------
# H1 known answers (the reference's own tests)
# ---------------------------------------------------------------------------
def test_h1_frozen(h1):
    d = dp()
    from paper_2604_14411_b200 import kernels as K

    assert h1.node_in.to_lists() == [[2], [0], [0, 1], []]
    assert h1.node_out.to_lists() == [[0], [1], [], [2]]
    assert h1.node_inc.to_lists() == [[0, 2], [0, 1], [0, 1], [2]]
    for rho, want in (([0, 0, 1, 1], 4.0), ([0, 1, 2, 3], 5.0), ([0, 1, 1, 0], 1.0), ([0, 0, 0, 0], 0.0)):
        assert d.connectivity(h1, d.Partitioning(np.array(rho), 4)) == want
    assert d.partition_sizes(h1, np.array([0, 0, 1, 1], np.int32), 2).tolist() == [2, 2]
    assert d.distinct_inbound_sizes(h1, np.array([0, 0, 1, 1], np.int32), 2).tolist() == [2, 2]
    assert d.materialize_neighbors(h1).to_lists() == [[1, 2, 3], [0, 2], [0, 1], [0]]
    assert K.resolve_matching(np.array([1, 0, 1]), np.array([5.0] * 3)).tolist() == [1, 0, 2]
    assert K.resolve_matching(np.array([1, 2, 1]), np.array([3.0, 7.0, 7.0])).tolist() == [0, 2, 1]
    with pytest.raises(d.MatchingInvariantError):
        K.resolve_matching(np.array([1, 2, 0]), np.ones(3))
    assert K.union_size_sorted(np.array([1, 4, 9]), np.array([4, 5])) == 4
    assert K.union_size_sorted(np.array([1, 4, 9]), np.zeros(0)) == 3
    part, st = d.partition(h1, d.Config(d.Constraints(2, 4)))
    assert part.assign.tolist() == [0, 1, 1, 0] and part.num_parts == 2 and st.num_partitions == 2
    assert st.levels == [{"nodes": 4, "edges": 3, "pins": 7}, {"nodes": 2, "edges": 3, "pins": 6}]
    assert st.connectivity_trace == [[1.0], [1.0]] and st.phase_ms == {}
    part, _ = d.partition(h1, d.Config(d.Constraints(4, 3)))
    assert part.num_parts == 1 and part.assign.tolist() == [0, 0, 0, 0]
    with pytest.raises(d.InfeasibleError, match="inbound"):
        d.partition(h1, d.Config(d.Constraints(4, 1)))
    with pytest.raises(d.InfeasibleError):
        d.partition(h1, d.Config(d.Constraints(0, 4)))
    with pytest.raises(d.InfeasibleError):
        d.partition(h1, d.Config(d.Constraints(4, -1)))
    assert d.check_validity(h1, d.Partitioning(np.array([0, 0, 0, 0]), 1), d.Constraints(2, 1)) == [
        d.Violation(0, "size", 4, 2), d.Violation(0, "inbound", 3, 1)]
    d.check_feasibility(h1, d.Constraints(1, 2))
    with pytest.raises(d.InfeasibleError):
        d.check_feasibility(h1, d.Constraints(1, 1))


# ---------------------------------------------------------------------------
# randomized parity vs the oracle, edge cases, errors
# ---------------------------------------------------------------------------
def test_random_instances_vs_oracle():
    rs = np.random.RandomState(113)
    for trial in range(30):
        n = int(rs.randint(5, 700))
        omega = int(rs.choice([2, 4, 8, 16, 32, 64]))
        g, c = make_instance(n, int(float(rs.choice([1.0, 1.5, 2.5])) * n), int(rs.choice([2, 3, 5, 8])),
                             seed=7000 + trial, omega=omega, delta_slack=int(rs.randint(0, 2 * omega)))
        assert_same_as_oracle(g, c.max_size, c.max_inbound)


def test_max_rounds_and_nonunit_node_sizes():
    d = dp()
    rs = np.random.RandomState(5)
    for trial in range(6):
        n = int(rs.randint(20, 300))
        g0, c = make_instance(n, 2 * n, 5, seed=9100 + trial, omega=32, delta_slack=20)
        sizes = rs.randint(1, 4, size=n).astype(np.int32)
        g = d.Hypergraph._from_csr(n, g0.edge_weight, g0.edge_src, g0.edge_dst, node_size=sizes)
        for rounds in (1, 3):
            assert_same_as_oracle(g, 32, c.max_inbound, max_rounds=rounds)


def test_layered_snn_vs_oracle():
    from paper_2604_14411_b200 import workloads as W

    for (layers, width, omega) in ((4, 256, 128), (6, 200, 256)):
        assert_same_as_oracle(graph(W.layered_snn(layers, width, fanout=32, window=128, seed=layers)), omega, 4096)


def test_power_law_vs_oracle():
    from paper_2604_14411_b200 import workloads as W

    arr = W.power_law(3000, 3000, k_max=300, seed=1)
    indeg = int(np.bincount(arr[5], minlength=3000).max())
    assert_same_as_oracle(graph(arr), 64, max(indeg, 256))


def test_degenerate_inputs():
    d = dp()
    # no edges: every node is its own part, connectivity 0
    g = d.Hypergraph._from_csr(5, np.zeros(0), d.CsrSets.from_lists([]), d.CsrSets.from_lists([]))
    part, st = d.partition(g, d.Config(d.Constraints(2, 0)))
    assert part.assign.tolist() == [0, 1, 2, 3, 4] and st.connectivity_trace == [[0.0]]
    # single-pin edges, a node on both sides, isolated nodes, zero weights
    g = d.Hypergraph.from_edges(6, [3.0, 1.0, 0.0, 2.0], [[0], [1], [], [2]], [[0], [], [3], [1, 0]])
    assert_same_as_oracle(g, 2, 3)
    assert_same_as_oracle(g, 6, 3)
    # empty graph
    g = d.Hypergraph._from_csr(0, np.zeros(0), d.CsrSets.from_lists([]), d.CsrSets.from_lists([]))
    part, st = d.partition(g, d.Config(d.Constraints(2, 0)))
    assert len(part.assign) == 0 and part.num_parts == 0 and st.num_partitions == 0


def test_max_levels_guard_message():
    d = dp()
    g, c = make_instance(60, 90, 4, seed=1, omega=8)
    with pytest.raises(d.DhgError, match="max_levels"):
        d.partition(g, d.Config(c, max_levels=1))


def test_dyadic_fractional_weights_bit_exact():
    """0.5- and 0.25-step weights (tests/golden/weights.npz, produced by the
    reference): exact after scaling by 2^S, so every payload is bit-exact."""
    z = load_npz("weights.npz")
    for t in z["cases"]:
        if str(z["kinds"][t]) in ("half", "quarter"):
            check_golden_case(z, t)


def test_decimal_weights_bit_exact():
    """0.1-step weights round at every f64 addition, so only the reference's
    own summation order reproduces its sums: the reference-order path
    (csrc/ordered.cuh) against every payload the reference recorded."""
    z = load_npz("weights.npz")
    for t in z["cases"]:
        if str(z["kinds"][t]) == "decimal":
            check_golden_case(z, t)


def test_feasibility_precedes_unsupported_input():
    """The reference checks feasibility first (driver.py:89): an infeasible
    graph with unsupported weights raises InfeasibleError, not DhgError."""
    d = dp()
    g = d.Hypergraph.from_edges(3, [0.1, 1.0], [[0], [1]], [[1, 2], [2]])
    with pytest.raises(d.InfeasibleError, match="inbound"):
        d.partition(g, d.Config(d.Constraints(2, 1)))


def test_observer_may_call_the_library():
    """An observer that evaluates the live payload objects (connectivity,
    sizes, validity) from inside the callback; the reference allows it."""
    d = dp()
    g, c = make_instance(300, 450, 5, seed=17, omega=8)
    seen = []

    def obs(kind, p):
        if kind == "level":
            co = p["coarse"]
            seen.append(("level", len(co.node_in.data), d.connectivity(co, d.Partitioning(
                np.arange(co.num_nodes, dtype=np.int32), co.num_nodes))))
        else:
            gr = p["graph"]
            part = d.Partitioning(p["assign"], p["num_parts"])
            seen.append(("round", d.connectivity(gr, part), len(d.check_validity(gr, part, c)) >= 0))

    part, st = d.partition(g, d.Config(c, max_levels=1 << 20), observer=obs)
    ref, _ = d.partition(g, d.Config(c, max_levels=1 << 20))
    assert np.array_equal(part.assign, ref.assign)
    assert any(k == "level" for k, *_ in seen) and any(k == "round" for k, *_ in seen)


def test_timings_and_determinism():
    d = dp()
    g, c = make_instance(400, 600, 5, seed=33, omega=8)
    p1, s1 = d.partition(g, d.Config(c))
    p2, s2 = d.partition(g, d.Config(c), timings=True)
    assert np.array_equal(p1.assign, p2.assign) and s1.levels == s2.levels
    assert set(s2.phase_ms) == {"coarsen", "refine", "total"} and all(v >= 0 for v in s2.phase_ms.values())


def test_driver_invariants_on_gpu_results():
    """The reference driver tests' properties, checked on the GPU result itself
    (pkg/tests/test_driver.py:60-121): valid and compacted, traces non-increasing
    within a level, strictly shrinking levels, final connectivity = trace end,
    observer counts, RunStats.to_dict shape."""
    d = dp()
    rs = np.random.RandomState(113)
    for trial in range(12):
        n = int(rs.randint(12, 300))
        omega = int(rs.choice([4, 8, 16]))
        g, c = make_instance(n, int(1.5 * n), 5, seed=1100 + trial, omega=omega, delta_slack=omega)
        seen = {"level": 0, "round": 0}

        def obs(kind, payload):
            seen[kind] += 1
            if kind == "level":
                assert payload["coarse"].num_nodes < payload["fine"].num_nodes
                assert payload["cmap"].num_coarse == payload["coarse"].num_nodes
            else:
                assert payload["selection"].k >= 0

        part, st = d.partition(g, d.Config(c), observer=obs)
        assert d.check_validity(g, part, c) == []
        assert np.unique(part.assign).tolist() == list(range(part.num_parts)) and st.num_partitions == part.num_parts
        for tr in st.connectivity_trace:
            assert all(b <= a for a, b in zip(tr, tr[1:]))
        sizes = [lv["nodes"] for lv in st.levels]
        assert all(b < a for a, b in zip(sizes, sizes[1:]))
        assert st.connectivity_trace[-1][-1] == d.connectivity(g, part)
        # a round is observed iff it proposed moves (refine.py:289-306): every
        # applied round was observed, and at most max_rounds per level
        applied = sum(len(tr) - 1 for tr in st.connectivity_trace)
        assert seen["level"] == len(st.levels) - 1 and applied <= seen["round"] <= 8 * len(st.levels)
        assert set(st.to_dict()) == {"levels", "connectivity_trace", "phase_ms", "num_partitions"}
    # the reference test's own instance (test_driver.py:97-111)
    g, c = make_instance(100, 150, 5, seed=47, omega=8)
    seen = {"level": 0, "round": 0}
    part, st = d.partition(g, d.Config(c), observer=lambda kind, _p: seen.__setitem__(kind, seen[kind] + 1))
    assert seen["level"] == len(st.levels) - 1 and seen["round"] >= len(st.levels)


def test_gpu_smoke_entry():
    import __graft_entry__

    __graft_entry__.smoke()


# ---------------------------------------------------------------------------
# full-size workload (C2): size-independent properties
# ---------------------------------------------------------------------------
def test_c2_full_size_properties():
    from paper_2604_14411_b200 import workloads as W

    d = dp()
    arrs, omega, delta, _ = W.make_config("C2")
    g = graph(arrs)
    p1, s1 = d.partition(g, d.Config(d.Constraints(omega, delta), max_levels=1 << 20))
    assert d.check_validity(g, p1, d.Constraints(omega, delta)) == []
    assert np.array_equal(np.unique(p1.assign), np.arange(p1.num_parts))
    assert s1.connectivity_trace[-1][-1] == d.connectivity(g, p1)
    for tr in s1.connectivity_trace:
        assert all(b <= a for a, b in zip(tr, tr[1:]))
    sizes = [lv["nodes"] for lv in s1.levels]
    assert all(b < a for a, b in zip(sizes, sizes[1:]))
    assert all(lv["edges"] == g.num_edges for lv in s1.levels)
    p2, s2 = d.partition(g, d.Config(d.Constraints(omega, delta), max_levels=1 << 20))
    assert np.array_equal(p1.assign, p2.assign) and s1.to_dict() == s2.to_dict()


_FORCED_TIERS_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from conftest import arrays_of, make_instance
from oracle import oracle as orc
import paper_2604_14411_b200 as dp
from paper_2604_14411_b200 import workloads as W
cases = []
rs = np.random.RandomState(77)
for t in range(8):
    n = int(rs.randint(50, 600))
    g, c = make_instance(n, 2 * n, int(rs.choice([3, 5, 8])), seed=8800 + t, omega=int(rs.choice([8, 32, 64])),
                         delta_slack=int(rs.randint(0, 40)))
    cases.append((g, c.max_size, c.max_inbound))
arr = W.power_law(1500, 1500, k_max=200, seed=3)
indeg = int(np.bincount(arr[5], minlength=1500).max())
n, w, so, sd, do, dd = arr
cases.append((dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd)), 128, max(indeg, 256)))
for g, om, de in cases:
    lev = []
    obs = lambda kind, p: lev.append(p) if kind == "level" else None
    part, st = dp.partition(g, dp.Config(dp.Constraints(om, de), max_levels=1 << 20), observer=obs)
    a, k, ost, oev = orc.partition(*arrays_of(g), g.node_size, max_size=om, max_inbound=de, max_levels=1 << 20,
                                   record=True)
    assert np.array_equal(part.assign, a), "assign differs"
    assert st.levels == ost["levels"] and st.connectivity_trace == ost["connectivity_trace"]
    olev = [e for e in oev if e["kind"] == "level"]
    assert len(olev) == len(lev)
    for e, o in zip(lev, olev):  # every level payload, the coarse graph's side order included
        f, cm, co = e["forest"], e["cmap"], e["coarse"]
        for got, key in ((f.pair, "pair"), (f.score, "score"), (f.match, "match"), (cm.gamma, "gamma"),
                         (co.edge_src.offsets, "src_off"), (co.edge_src.data, "src_dat"),
                         (co.edge_dst.offsets, "dst_off"), (co.edge_dst.data, "dst_dat"),
                         (co.node_size, "node_size")):
            assert np.array_equal(got, o[key]), ("level payload differs", e["index"], key)
print("forced tiers ok", len(cases))
"""


def test_every_kernel_tier_under_forced_escalation():
    """DHGP_FORCE_TIERS=1 shrinks the warp/block escalation thresholds so that
    the medium, block and dense tiers of scoring and proposing all run;
    DHGP_KEEP_LEVELS_BYTES=0 forces the checkpoint + rebuild path for every
    level that is not a checkpoint."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    for mode in ("1", "2"):  # 1: medium + block tiers; 2: the small-K dense path
        r = subprocess.run([sys.executable, "-c", _FORCED_TIERS_SCRIPT, root], capture_output=True, text=True,
                           env=dict(os.environ, DHGP_FORCE_TIERS=mode, DHGP_KEEP_LEVELS_BYTES="0"), timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
        assert "forced tiers ok" in r.stdout


def test_c2_stepwise_levels_match_oracle():
    """Full-size C2 (the bench workload): sampled coarsening and refinement
    levels of one GPU run replayed by the oracle (tests/stepwise_parity.py)."""
    import stepwise_parity as sp

    out = sp.check_config("C2", [990], [0, 900])
    assert len(out["coarsen"]) == 1 and len(out["refine"]) >= 1
    assert all(r["bit_exact"] for r in out["coarsen"] + out["refine"]), out


def test_full_and_incremental_paths_agree(monkeypatch):
    """DHGP_FULL_REFINE=1 / DHGP_FULL_SCORE=1 recompute every run list,
    proposal and candidate score on every round / level (the direct
    restatement); the default incremental paths recompute only what moves,
    projections and merges dirtied.  Both must equal the oracle, and on the
    full-size C2 workload each other."""
    from paper_2604_14411_b200 import workloads as W

    rs = np.random.RandomState(4242)
    cases = []
    for t in range(10):
        n = int(rs.randint(30, 900))
        g, c = make_instance(n, int(rs.choice([1, 2, 3])) * n, int(rs.choice([3, 5, 8])), seed=6100 + t,
                             omega=int(rs.choice([4, 16, 64])), delta_slack=int(rs.randint(0, 30)))
        cases.append((g, c.max_size, c.max_inbound, int(rs.choice([1, 2, 8]))))
    cases.append((graph(W.layered_snn(5, 300, fanout=32, window=96, seed=9)), 256, 4096, 8))
    cases.append((graph(W.layered_snn(8, 400, fanout=48, window=128, seed=3)), 512, 1024, 8))
    arr = W.power_law(2500, 2500, k_max=400, seed=11)  # h-edges over 128 pins: the block run-list update
    cases.append((graph(arr), 64, max(int(np.bincount(arr[5], minlength=2500).max()), 256), 8))
    for mode in ("1", "0"):
        monkeypatch.setenv("DHGP_FULL_REFINE", mode)
        monkeypatch.setenv("DHGP_FULL_SCORE", mode)
        for g, om, de, mr in cases:
            assert_same_as_oracle(g, om, de, max_rounds=mr)
    arrs, om, de, _ = W.make_config("C2")
    g = graph(arrs)
    res = []
    for mode in ("1", "0"):
        monkeypatch.setenv("DHGP_FULL_REFINE", mode)
        monkeypatch.setenv("DHGP_FULL_SCORE", mode)
        res.append(run_gpu(g, om, de, max_levels=1 << 20)[:2])
    (p1, s1), (p2, s2) = res
    assert np.array_equal(p1.assign, p2.assign) and s1.to_dict() == s2.to_dict()


def test_connectivity_exact_for_any_weights():
    """connectivity() (dhgp_evaluate) and the connectivity_value seam equal the
    reference's ascending-edge f64 sum (_kernels.pyx:199-213, via the pinned
    oracle) for integral, dyadic and decimal weights alike: a parallel int64
    sum when it is provably exact, else the ordered walk."""
    d = dp()
    from paper_2604_14411_b200 import kernels as K

    rs = np.random.RandomState(99)
    for t, scale in enumerate((1.0, 0.5, 0.125, 0.1, 1e-3, 3.0e15)):
        g, c = make_instance(500, 800, 6, seed=200 + t, omega=8)
        w = rs.randint(1, 50, size=g.num_edges) * scale
        g = d.Hypergraph._from_csr(g.num_nodes, w, g.edge_src, g.edge_dst)
        a = rs.randint(0, 37, size=g.num_nodes).astype(np.int32)
        want = orc.connectivity_value(g.edge_pins.offsets, g.edge_pins.data, w, a)
        assert d.connectivity(g, d.Partitioning(a, 37)) == want, scale
        assert K.connectivity_value(g.edge_pins.offsets, g.edge_pins.data, w, a) == want, scale


def test_hedge_beyond_shared_memory_golden():
    """One h-edge of 8,300 pins (more than the 8,192 slots a per-segment sort
    or a wide run update keeps in shared memory): the global-memory paths,
    bit-exact against the reference's own partition (tests/golden/bigedge.npz)."""
    z = load_npz("bigedge.npz")
    g = graph([z[f"in_{k}"] for k in ("n", "w", "so", "sd", "do", "dd")])
    assert int(np.diff(g.edge_pins.offsets).max()) > 8192
    part, st, _ = run_gpu(g, int(z["omega"]), int(z["delta"]), max_levels=1 << 20)
    ref = json.loads(bytes(z["stats"]).decode())
    assert np.array_equal(part.assign, z["assign"]) and part.num_parts == int(z["num_parts"])
    assert st.levels == ref["levels"] and st.connectivity_trace == ref["trace"]


def test_c2_whole_run_matches_reference():
    """C2 (100k-node layered SNN, the reference's 9,755 s single-core run,
    tests/golden/make_c2_golden.py): the GPU partition's assignment, part
    count, every level's sizes and the whole connectivity trace equal the
    reference's (driver.py:76-163 end to end)."""
    from paper_2604_14411_b200 import workloads as W

    z = load_npz("c2.npz")
    meta = json.loads(bytes(z["meta"]).decode())
    arrs, omega, delta, _ = W.make_config("C2")
    g = graph(arrs)
    part, st, _ = run_gpu(g, omega, delta, max_levels=1 << 20)
    ref = json.loads(bytes(z["stats"]).decode())
    assert (omega, delta) == (meta["omega"], meta["delta"])
    assert np.array_equal(part.assign, z["assign"]) and part.num_parts == int(z["num_parts"])
    assert st.levels == ref["levels"]
    assert st.connectivity_trace == ref["trace"]
