"""Diagnostics: per-scope timing histogram of one warm partition (default C2; DHGP_TRACE=1)."""
import os, subprocess, sys, collections
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if os.environ.get("DHGP_TRACE") != "1":
    env = dict(os.environ, DHGP_TRACE="1")
    r = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    if os.environ.get("DHGP_TRACE_RAW"):
        with open(os.environ["DHGP_TRACE_RAW"], "w") as f:
            f.write(r.stdout + r.stderr)
    agg = collections.defaultdict(lambda: [0, 0.0, []])
    err = r.stderr.split("=== WARM ===")[-1]  # the second (warm) partition only
    for ln in err.splitlines():
        if ln.startswith("trace "):
            _, nm, ms, tag = ln.split()
            a = agg[nm]; a[0] += 1; a[1] += float(ms); a[2].append((float(ms), int(tag)))
    print(r.stdout[-2000:])
    for nm, (n, tot, lst) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lst.sort(reverse=True)
        print(f"{nm:14s} n={n:6d} total={tot:9.1f} ms  top={[(round(m,2), t) for m, t in lst[:6]]}")
        # by size bucket of the tag (N)
        b = collections.defaultdict(lambda: [0, 0.0])
        for m, t in lst:
            k = 0 if t < 0 else len(str(t))
            b[k][0] += 1; b[k][1] += m
        print("      by digits of N:", {k: (v[0], round(v[1], 1)) for k, v in sorted(b.items())})
    sys.exit(0)
sys.path.insert(0, ROOT)
import paper_2604_14411_b200 as dp
from paper_2604_14411_b200 import workloads as W
arrs, om, de, _ = W.make_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
n, w, so, sd, do, dd = arrs
g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
import time
dp.partition(g, dp.Config(dp.Constraints(om, de), max_levels=1 << 20))  # warm-up (allocator, module load)
print("=== WARM ===", file=sys.stderr, flush=True)
t = time.perf_counter()
p, s = dp.partition(g, dp.Config(dp.Constraints(om, de), max_levels=1 << 20))
print("total", time.perf_counter() - t, len(s.levels), p.num_parts)
import json
print("LEVELS", json.dumps(s.levels))
print("TRACE", json.dumps([len(t) for t in s.connectivity_trace]))
