"""Diagnostics: time the GPU .dhg parser against the host restatement of the
reference's parse_dhg on a config's text (written once with numpy).

    python tests/parse_probe.py C5 [--host]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_14411_b200 as dp  # noqa: E402
from paper_2604_14411_b200 import workloads as W  # noqa: E402


def dhg_text_fast(n, w, so, sd, do, dd) -> str:
    """Same bytes as workloads.dhg_text for integral weights, built per column."""
    E = len(w)
    ks, kd = np.diff(so), np.diff(do)
    # one token list per line: w ks kd src... dst...
    cnt = 3 + ks + kd
    tok = np.empty(int(cnt.sum()), dtype=np.int64)
    start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    tok[start] = w.astype(np.int64)
    tok[start + 1] = ks
    tok[start + 2] = kd
    # pins: positions start+3 .. within each line
    line_of_src = np.repeat(np.arange(E), ks)
    pos_src = start[line_of_src] + 3 + (np.arange(len(sd)) - so[line_of_src])
    tok[pos_src] = sd
    line_of_dst = np.repeat(np.arange(E), kd)
    pos_dst = start[line_of_dst] + 3 + ks[line_of_dst] + (np.arange(len(dd)) - do[line_of_dst])
    tok[pos_dst] = dd
    s = tok.astype(str)
    sep = np.full(len(tok), " ", dtype=object)
    sep[np.cumsum(cnt) - 1] = "\n"
    body = "".join(np.char.add(s, sep.astype(str)).tolist())
    return f"{E} {n}\n" + body


name = sys.argv[1] if len(sys.argv) > 1 else "C5"
arrs, _, _, desc = W.make_config(name)
t = time.perf_counter()
text = dhg_text_fast(*arrs)
gen = time.perf_counter() - t
dp.parse_dhg("1 2\n1 1 1 0 1\n")  # context warm-up
ts = []
for _ in range(3):
    t = time.perf_counter()
    g = dp.parse_dhg(text)
    ts.append(time.perf_counter() - t)
out = {"config": name, "bytes": len(text), "edges": g.num_edges, "pins": g.num_pins(), "text_build_s": round(gen, 2),
       "gpu_parse_s": round(min(ts), 4), "gpu_parse_GBps_e2e": round(len(text) / min(ts) / 1e9, 3)}
n, w, so, sd, do, dd = arrs
assert np.array_equal(g.edge_src.data, sd) and np.array_equal(g.edge_dst.data, dd) and np.array_equal(g.edge_weight, w)
if "--host" in sys.argv:
    t = time.perf_counter()
    h = dp.parse_dhg_host(text)
    out["host_parse_s"] = round(time.perf_counter() - t, 2)
    out["speedup"] = round(out["host_parse_s"] / out["gpu_parse_s"], 1)
print(json.dumps(out))
