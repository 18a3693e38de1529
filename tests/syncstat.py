"""Diagnostics: host time blocked in syncs vs wall time (DHGP_SYNCSTAT=1), plus
the scoring-tier counters of DHGP_TRACE=1 when that is set.  Usage:
DHGP_SYNCSTAT=1 python tests/syncstat.py C2 [repeats]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_14411_b200 as dp
from paper_2604_14411_b200 import workloads as W
arrs, om, de, _ = W.make_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
n, w, so, sd, do, dd = arrs
g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    p, s = dp.partition(g, dp.Config(dp.Constraints(om, de), max_levels=1 << 20))
