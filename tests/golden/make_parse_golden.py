"""Golden vectors for the .dhg text format, produced by the REFERENCE's own
parse_dhg (hgraph.py:409-467) — run in the build container, where
/root/reference is importable:

    python tests/golden/make_parse_golden.py   # writes tests/golden/parse_cases.json

Each case: the text, and either the parsed primary arrays or the exception
class, line and message.  tests/ check the host restatement (CPU tier) and
the GPU parser (gpu tier) against these.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import dhgpart  # noqa: E402
from dhgpart import hgraph  # noqa: E402

H1 = "3 4\n1 1 2 0 1 2\n2 1 1 1 2\n1 1 1 3 0\n"
CASES = [
    H1, H1.rstrip("\n"), H1 + "\n\n   \n\t\n", H1.replace("\n", "\r\n"), H1.replace(" ", "\t"),
    "", "\n", "  \n\n", "0 5\n", "0 5", "0 0\n", "3\n", "3 4 5\n", "a 4\n", "-1 4\n", "1 -4\n",
    "3 4\n1 1 2 0 1 2\n", "1 4\n1 1 2 0 1 2\n2 1 1 1 2\n", "2 3\n\n1 1 1 0 1\n",
    "1 3\n1 1\n", "1 3\nx 1 1 0 1\n", "1 3\n1 1.5 1 0 1\n", "1 3\n-1 1 1 0 1\n", "1 3\ninf 1 1 0 1\n",
    "1 3\nnan 1 1 0 1\n", "1 3\n1 0 0\n", "1 3\n1 -1 2 0 1\n", "1 3\n1 1 1 0\n", "1 3\n1 1 1 0 1 2\n",
    "1 3\n1 1 1 0 x\n", "1 3\n1 1 1 0 3\n", "1 3\n1 1 1 0 -1\n", "1 3\n1 2 1 0 0 1\n", "1 3\n1 1 2 0 1 1\n",
    "1 3\n1 1 1 1 1\n", "1 3\n2.5 1 1 0 1\n", "1 3\n1e1 1 1 0 1\n", "1 3\n+3 +1 1 0 +2\n", "1 3\n1_0 1 1 0 1_0\n",
    "1 3\n007 01 01 00 02\n", "1 3\n1 1 1 0 1\x1c\n", "1 3\n1 1 1 0\xa01\n", "1 3\n1 1 1 ١ 2\n",
    "2 10\n1 1 1 0 1\n2 1 1 0 99\n", "3 10\n1 1 1 0 1\n1 1 1 0 99\n1 1 1 5 5 5\n",
    "2 10\n1 1 1 0 1.5\n1 1 1 0 99\n", "2 10\n1 1 1 0 1\n1 1 1 0\n", "2 5\n1 1 1 4 4\n9 2 0 3 1\n",
    "1 3\n99999999999999999999 1 1 0 1\n", "1 3\n1 1 1 000000000000000000001 2\n",
    "1 3\n1 99999999999 1 0 1\n",
]


def run(text):
    try:
        g = hgraph.parse_dhg(text)
        return {"text": text, "ok": True, "num_nodes": g.num_nodes, "weights": g.edge_weight.tolist(),
                "src_off": g.edge_src.offsets.tolist(), "src_dat": g.edge_src.data.tolist(),
                "dst_off": g.edge_dst.offsets.tolist(), "dst_dat": g.edge_dst.data.tolist()}
    except Exception as ex:  # noqa: BLE001 — the golden records any exception
        return {"text": text, "ok": False, "exc": type(ex).__name__, "line": getattr(ex, "line", None),
                "msg": str(ex)}


if __name__ == "__main__":
    out = [run(t) for t in CASES]
    Path(__file__).with_name("parse_cases.json").write_text(json.dumps(out, indent=0))
    print(len(out), "cases;", sum(1 for o in out if o["ok"]), "parse")
