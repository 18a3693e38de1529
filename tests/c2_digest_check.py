"""Level-by-level and round-by-round parity of a GPU partition against the
reference's own whole-run record (tests/golden/c2_levels.jsonl.gz, written by
tests/golden/make_c2_golden.py from oracle/_ref): the same sha1 digests of
every observer payload — pair, score, match, gamma and the coarse graph per
coarsening level; assign, moves, gain_iso, gain_seq, active, k, total_gain
per refinement round.  Run on the GPU box:

    python tests/c2_digest_check.py [--config C2] [--json out.json]

Test infrastructure (imports no oracle; reads only the committed golden).
"""
from __future__ import annotations

import argparse
import gzip
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))

from make_c2_golden import digest  # noqa: E402  (the same digest function)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--golden", default=str(ROOT / "tests" / "golden" / "c2_levels.jsonl.gz"))
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    import paper_2604_14411_b200 as dp
    from paper_2604_14411_b200 import workloads as W

    ref = [json.loads(ln) for ln in gzip.open(a.golden, "rt")]
    arrs, omega, delta, _ = W.make_config(a.config)
    n, w, so, sd, do, dd = arrs
    g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
    got = []

    def obs(kind, p):
        if kind == "level":
            f, c, cm = p["forest"], p["coarse"], p["cmap"]
            got.append({"kind": "level", "index": p["index"], "pair": digest(f.pair), "score": digest(f.score),
                        "match": digest(f.match), "gamma": digest(cm.gamma),
                        "coarse": digest(c.edge_src.offsets, c.edge_src.data, c.edge_dst.offsets, c.edge_dst.data,
                                         c.node_size)})
        else:
            m, s = p["moves"], p["selection"]
            got.append({"kind": "round", "level": p["level"], "round": p["round"], "assign": digest(p["assign"]),
                        "mv": digest(m.node, m.from_part, m.to_part), "gain_iso": digest(m.gain_iso),
                        "gain_seq": digest(m.gain_seq), "active": digest(s.active), "k": int(s.k),
                        "total_gain": float(s.total_gain)})

    t = time.time()
    dp.partition(g, dp.Config(dp.Constraints(omega, delta), max_levels=1 << 20), observer=obs)
    keys = {"level": ("index", "pair", "score", "match", "gamma", "coarse"),
            "round": ("level", "round", "assign", "mv", "gain_iso", "gain_seq", "active", "k", "total_gain")}
    first_bad = None
    for i, (r, m) in enumerate(zip(ref, got)):
        if r["kind"] != m["kind"] or any(r[k] != m[k] for k in keys[r["kind"]]):
            first_bad = {"event": i, "reference": r, "gpu": m}
            break
    out = {"config": a.config, "events_reference": len(ref), "events_gpu": len(got),
           "levels": sum(1 for r in ref if r["kind"] == "level"), "rounds": sum(1 for r in ref if r["kind"] == "round"),
           "all_equal": first_bad is None and len(ref) == len(got), "first_difference": first_bad,
           "gpu_run_with_observer_s": round(time.time() - t, 1)}
    print(json.dumps(out))
    if a.json:
        Path(a.json).write_text(json.dumps(out, indent=1))
    sys.exit(0 if out["all_equal"] else 1)


if __name__ == "__main__":
    main()
