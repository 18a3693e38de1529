"""One partition of a workload config (default C2) for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_14411_b200 as dp
from paper_2604_14411_b200 import workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
arrs, om, de, _ = W.make_config(name)
n, w, so, sd, do, dd = arrs
g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
p, s = dp.partition(g, dp.Config(dp.Constraints(om, de), max_levels=1 << 20))
print("levels", len(s.levels), "parts", p.num_parts, "conn", s.connectivity_trace[-1][-1])
