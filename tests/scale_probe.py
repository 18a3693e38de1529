"""Diagnostics: time one partition of a workload config through the public API
and print a JSON line (levels, parts, connectivity, phases, launches).

    python tests/scale_probe.py C3 [--repeat R]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_14411_b200 as dp  # noqa: E402
from paper_2604_14411_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
repeat = int(sys.argv[sys.argv.index("--repeat") + 1]) if "--repeat" in sys.argv else 1
t0 = time.perf_counter()
arrs, om, de, desc = W.make_config(name)
n, w, so, sd, do, dd = arrs
g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
gen_s = time.perf_counter() - t0
for r in range(repeat):
    t = time.perf_counter()
    p, s = dp.partition(g, dp.Config(dp.Constraints(om, de), max_levels=1 << 20), timings=True)
    el = time.perf_counter() - t
    print(json.dumps({"config": name, "desc": desc, "gen_s": round(gen_s, 2), "e2e_s": round(el, 4),
                      "nodes": int(n), "h_edges": int(len(w)), "pins": int(len(sd) + len(dd)),
                      "max_size": om, "max_inbound": de, "levels": len(s.levels), "parts": p.num_parts,
                      "connectivity": s.connectivity_trace[-1][-1] if s.connectivity_trace else None,
                      "phase_ms": s.phase_ms, "launches": getattr(s, "_gpu_launches", None)}), flush=True)
    if "--levels" in sys.argv:
        with open(sys.argv[sys.argv.index("--levels") + 1], "w") as f:
            json.dump({"levels": s.levels, "rounds": [len(t) for t in s.connectivity_trace]}, f)
