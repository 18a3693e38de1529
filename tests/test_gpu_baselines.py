"""GPU comparison baselines (csrc/baselines.cu) against the reference's own
one_pass / overlap_greedy (baselines.py:16-91): bit-identical assignments and
partition counts on the golden fixtures (tests/golden/make_baseline_golden.py),
validity at the bench scale, and the reference's error behaviour."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import H1_TEXT, load_npz

pytestmark = pytest.mark.gpu


def dp():
    import paper_2604_14411_b200 as m

    return m


def test_baselines_match_reference_fixtures():
    d = dp()
    z = load_npz("baselines.npz")
    for i in z["cases"]:
        p = f"c{i}_"
        n, w, so, sd, do, dd = (z[f"{p}in_{k}"] for k in ("n", "w", "so", "sd", "do", "dd"))
        g = d.Hypergraph._from_csr(int(n), w, d.CsrSets(so, sd), d.CsrSets(do, dd), node_size=z[p + "size"])
        c = d.Constraints(int(z[p + "omega"]), int(z[p + "delta"]))
        a = d.one_pass(g, c)
        assert np.array_equal(a.assign, z[p + "onepass"]) and a.num_parts == int(z[p + "onepass_k"]), i
        b = d.overlap_greedy(g, c)
        assert np.array_equal(b.assign, z[p + "overlap"]) and b.num_parts == int(z[p + "overlap_k"]), i
        assert not d.check_validity(g, a, c) and not d.check_validity(g, b, c)


def test_baselines_on_h1_and_errors():
    d = dp()
    g = d.parse_dhg_host(H1_TEXT)
    # H1 with generous limits: one_pass keeps everything in one partition
    p = d.one_pass(g, d.Constraints(4, 3))
    assert p.num_parts == 1 and p.assign.tolist() == [0, 0, 0, 0]
    with pytest.raises(d.InfeasibleError):
        d.one_pass(g, d.Constraints(2, 1))  # node 2 has 2 inbound h-edges
    with pytest.raises(d.InfeasibleError):
        d.overlap_greedy(g, d.Constraints(0, 4))


def test_baselines_at_bench_scale_are_valid_and_deterministic():
    from paper_2604_14411_b200 import workloads as W

    d = dp()
    arrs, om, de, _ = W.make_config("C2")
    n, w, so, sd, do, dd = arrs
    g = d.Hypergraph._from_csr(n, w, d.CsrSets(so, sd), d.CsrSets(do, dd))
    c = d.Constraints(om, de)
    for fn in (d.one_pass, d.overlap_greedy):
        a, b = fn(g, c), fn(g, c)
        assert np.array_equal(a.assign, b.assign) and a.num_parts == b.num_parts
        assert not d.check_validity(g, a, c)
