#!/bin/bash
# compute-sanitizer evidence: memcheck / racecheck / synccheck /
# initcheck over the partition path, on the GPU box.  Logs -> gpurun_out/.
#   memcheck, initcheck: C1 (gen.py 10k / 20k) through partition();
#   racecheck, synccheck: a small instance under DHGP_FORCE_TIERS=1 and =2
#     (every kernel tier, the shared-memory hash tables, the CTA-pair DSMEM
#     merge, the global-memory sort / mover paths) — racecheck instruments
#     every shared-memory access, so the instance is kept small.
set -u
O=gpurun_out
mkdir -p $O
CS=compute-sanitizer
RUN_C1='import sys; sys.path.insert(0, "."); import paper_2604_14411_b200 as dp; from paper_2604_14411_b200 import workloads as W
a, om, de, _ = W.make_config("C1"); n, w, so, sd, do, dd = a
g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
p, s = dp.partition(g, dp.Config(dp.Constraints(om, de), max_levels=1 << 20)); print("C1", p.num_parts, s.connectivity_trace[-1][-1])'
RUN_SMALL='import sys; sys.path.insert(0, "."); import numpy as np, paper_2604_14411_b200 as dp; from paper_2604_14411_b200 import workloads as W
for seed, (nn, mp, om) in enumerate([(300, 5, 8), (500, 8, 32)]):
    n, w, so, sd, do, dd = W.random_dhg(nn, 2 * nn, mp, seed=40 + seed)
    g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
    de = int(np.bincount(dd, minlength=n).max()) + 4
    p, s = dp.partition(g, dp.Config(dp.Constraints(om, de), max_levels=1 << 20)); print("small", p.num_parts)
n, w, so, sd, do, dd = W.power_law(600, 600, k_max=150, seed=3)
g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
de = max(int(np.bincount(dd, minlength=n).max()), 256)
p, s = dp.partition(g, dp.Config(dp.Constraints(64, de), max_levels=1 << 20)); print("powerlaw", p.num_parts)'
$CS --tool memcheck --leak-check no --error-exitcode 9 python -c "$RUN_C1" > $O/sanitizer_memcheck_C1.log 2>&1; echo "memcheck rc=$?" >> $O/sanitizer_memcheck_C1.log
$CS --tool initcheck --error-exitcode 9 python -c "$RUN_C1" > $O/sanitizer_initcheck_C1.log 2>&1; echo "initcheck rc=$?" >> $O/sanitizer_initcheck_C1.log
for t in 1 2; do
  DHGP_FORCE_TIERS=$t DHGP_KEEP_LEVELS_BYTES=0 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python -c "$RUN_SMALL" > $O/sanitizer_racecheck_tiers$t.log 2>&1; echo "racecheck rc=$?" >> $O/sanitizer_racecheck_tiers$t.log
  DHGP_FORCE_TIERS=$t $CS --tool synccheck --error-exitcode 9 python -c "$RUN_SMALL" > $O/sanitizer_synccheck_tiers$t.log 2>&1; echo "synccheck rc=$?" >> $O/sanitizer_synccheck_tiers$t.log
  DHGP_FORCE_TIERS=$t $CS --tool memcheck --leak-check no --error-exitcode 9 python -c "$RUN_SMALL" > $O/sanitizer_memcheck_tiers$t.log 2>&1; echo "memcheck rc=$?" >> $O/sanitizer_memcheck_tiers$t.log
done
tail -n 3 $O/sanitizer_*.log
