"""Diagnostics for A/B kernel changes: time a config through the public API
(best of R) and print the sha1 of the assignment, the level sizes and the
connectivity trace, so two builds / env settings can be compared bit for bit.

    python tests/ab_probe.py C3 [R]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_14411_b200 as dp  # noqa: E402
from paper_2604_14411_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
arrs, om, de, _ = W.make_config(name)
n, w, so, sd, do, dd = arrs
g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
cfg = dp.Config(dp.Constraints(om, de), max_levels=1 << 20)
ts = []
for _ in range(reps):
    t = time.perf_counter()
    p, s = dp.partition(g, cfg)
    ts.append(time.perf_counter() - t)
h = hashlib.sha1()
h.update(np.ascontiguousarray(p.assign).tobytes())
h.update(json.dumps(s.levels).encode())
h.update(json.dumps(s.connectivity_trace).encode())
print(json.dumps({"config": name, "env": {k: v for k, v in os.environ.items() if k.startswith("DHGP_")},
                  "best_s": round(min(ts), 4), "all_s": [round(x, 4) for x in ts], "parts": p.num_parts,
                  "connectivity": s.connectivity_trace[-1][-1], "sha1": h.hexdigest()}), flush=True)
