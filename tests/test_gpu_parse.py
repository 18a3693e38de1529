"""The .dhg parser on the GPU against the reference's
golden cases and against the host restatement on large generated texts,
including lines that take the host path and errors far into the file."""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.num_nodes == b.num_nodes
    assert np.array_equal(a.edge_weight, b.edge_weight)
    for x, y in ((a.edge_src, b.edge_src), (a.edge_dst, b.edge_dst)):
        assert np.array_equal(x.offsets, y.offsets) and np.array_equal(x.data, y.data)


def test_reference_golden_cases():
    import paper_2604_14411_b200 as dp

    for case in json.loads((ROOT / "tests" / "golden" / "parse_cases.json").read_text()):
        if case["ok"]:
            g = dp.parse_dhg(case["text"])
            assert g.num_nodes == case["num_nodes"], case["text"]
            assert g.edge_weight.tolist() == case["weights"], case["text"]
            assert g.edge_src.offsets.tolist() == case["src_off"] and g.edge_src.data.tolist() == case["src_dat"]
            assert g.edge_dst.offsets.tolist() == case["dst_off"] and g.edge_dst.data.tolist() == case["dst_dat"]
        else:
            with pytest.raises(dp.DhgParseError) as ei:
                dp.parse_dhg(case["text"])
            assert (str(ei.value), ei.value.line) == (case["msg"], case["line"]), case["text"]


def _big_text(seed=3, n=12000, m=20000):
    from paper_2604_14411_b200 import workloads as W

    arr = W.random_dhg(n, m, 9, seed=seed)
    return W.dhg_text(*arr)


def test_large_text_matches_host_including_host_path_lines():
    import paper_2604_14411_b200 as dp

    text = _big_text()
    _same(dp.parse_dhg(text), dp.parse_dhg_host(text))
    lines = text.split("\n")
    rs = np.random.RandomState(1)
    for i in rs.choice(np.arange(1, len(lines) - 1), 300, replace=False):
        tok = lines[i].split()
        k = int(rs.randint(5))
        if k == 0:
            tok[0] = tok[0] + ".25"          # decimal weight
        elif k == 1:
            tok[1] = "+" + tok[1]            # signed count
        elif k == 2:
            tok[-1] = "0" * 12 + tok[-1]     # long literal with leading zeros
        elif k == 3:
            lines[i] = "\u00a0".join(tok)  # non-ASCII separator
            continue
        else:
            lines[i] = "\t ".join(tok) + " \r"  # other ASCII whitespace
            continue
        lines[i] = " ".join(tok)
    text2 = "\n".join(lines) + "\n \n\n"
    _same(dp.parse_dhg(text2), dp.parse_dhg_host(text2))


@pytest.mark.parametrize("kind", ["range", "dup", "count", "weight", "slow_first"])
def test_first_error_far_into_the_file(kind):
    import paper_2604_14411_b200 as dp

    lines = _big_text(seed=5).split("\n")
    a, b = 15001, 17002  # two bad lines: the first one must be reported
    for i in (a, b):
        tok = lines[i].split()
        ks = int(tok[1])
        if kind == "range":
            tok[-1] = "99999999"
        elif kind == "dup":
            if ks >= 2:
                tok[4] = tok[3]
            else:
                tok = [tok[0], "2", "0", "7", "7"]
        elif kind == "count":
            tok = tok[:-1]
        elif kind == "weight":
            tok[0] = "-2"
        elif kind == "slow_first":
            tok[0] = "nan" if i == a else tok[0]
            if i == b:
                tok[-1] = "99999999"
        lines[i] = " ".join(tok)
    text = "\n".join(lines)
    with pytest.raises(dp.DhgParseError) as e_gpu:
        dp.parse_dhg(text)
    with pytest.raises(dp.DhgParseError) as e_host:
        dp.parse_dhg_host(text)
    assert (str(e_gpu.value), e_gpu.value.line) == (str(e_host.value), e_host.value.line)
    assert e_gpu.value.line == a + 1


def test_parsed_graph_partitions_like_the_host_parsed_one():
    import paper_2604_14411_b200 as dp

    text = _big_text(seed=9, n=3000, m=5000)
    c = dp.Config(dp.Constraints(64, 400), max_levels=1 << 20)
    p1, s1 = dp.partition(dp.parse_dhg(text), c)
    p2, s2 = dp.partition(dp.parse_dhg_host(text), c)
    assert np.array_equal(p1.assign, p2.assign) and s1.connectivity_trace == s2.connectivity_trace
