"""Whole-run golden for C2 from the REFERENCE itself (oracle/_ref, the
unmodified dhgpart package with its compiled backend), run to completion on
one host core.  Run here, where /root/reference exists (hours):

    python tests/golden/make_c2_golden.py [--config C2] [--out tests/golden/c2.npz]

Writes, incrementally (so a killed run keeps what it reached):
  <out>.levels.jsonl — one line per coarsening level: wall time since start,
                       the level's seconds, node/pin counts, and sha1 digests
                       of the observer payload (pair, score, match, gamma and
                       the coarse graph's five arrays);
                       one line per refinement round: level, round, seconds,
                       digests of (assign, moves, gain_iso, gain_seq, active),
                       k and total_gain.
  <out>              — final assign, num_parts, RunStats (levels, trace),
                       total seconds and the host description.

The per-level digests let tests/diag_parity.py name the first differing level
of a GPU run without storing 1000 levels of arrays.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref_loader  # noqa: E402
from paper_2604_14411_b200 import workloads as W  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha1()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(np.int64(a.size).tobytes())
        h.update(a.tobytes())
    return h.hexdigest()[:16]


def host_desc() -> str:
    try:
        cpu = [ln.split(":", 1)[1].strip() for ln in subprocess.run(
            ["lscpu"], capture_output=True, text=True).stdout.splitlines() if ln.startswith("Model name")][0]
    except Exception:
        cpu = platform.processor()
    return f"{cpu}; {os.cpu_count()} logical cpus; 1 core used (the reference is single-threaded)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--out", default=str(ROOT / "tests" / "golden" / "c2.npz"))
    a = ap.parse_args()
    dp = ref_loader.load()
    arrs, omega, delta, desc = W.make_config(a.config)
    n, w, so, sd, do, dd = arrs
    g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
    log = open(a.out + ".levels.jsonl", "w")
    t_start = time.perf_counter()
    last = [t_start]

    def stamp():
        now = time.perf_counter()
        dt, last[0] = now - last[0], now
        return round(now - t_start, 3), round(dt, 3)

    def obs(kind, p):
        t, dt = stamp()
        if kind == "level":
            f, c, cm = p["forest"], p["coarse"], p["cmap"]
            rec = {"kind": "level", "index": p["index"], "t": t, "dt": dt, "nodes": int(p["fine"].num_nodes),
                   "pins": int(p["fine"].num_pins()), "coarse_nodes": int(c.num_nodes),
                   "pair": digest(f.pair), "score": digest(f.score), "match": digest(f.match),
                   "gamma": digest(cm.gamma),
                   "coarse": digest(c.edge_src.offsets, c.edge_src.data, c.edge_dst.offsets, c.edge_dst.data,
                                    c.node_size)}
        else:
            m, s = p["moves"], p["selection"]
            rec = {"kind": "round", "level": p["level"], "round": p["round"], "t": t, "dt": dt,
                   "moves": int(len(m.node)), "assign": digest(p["assign"]),
                   "mv": digest(m.node, m.from_part, m.to_part), "gain_iso": digest(m.gain_iso),
                   "gain_seq": digest(m.gain_seq), "active": digest(s.active), "k": int(s.k),
                   "total_gain": float(s.total_gain)}
        log.write(json.dumps(rec) + "\n")
        log.flush()

    cfg = dp.Config(dp.Constraints(omega, delta), max_levels=1 << 20)
    part, st = dp.partition(g, cfg, observer=obs, timings=True)
    total = time.perf_counter() - t_start
    log.close()
    np.savez_compressed(
        a.out, assign=part.assign, num_parts=np.int64(part.num_parts),
        stats=np.frombuffer(json.dumps({"levels": st.levels, "trace": st.connectivity_trace}).encode(), np.uint8),
        meta=np.frombuffer(json.dumps({"config": a.config, "desc": desc, "omega": omega, "delta": delta,
                                       "seconds": total, "phase_ms": st.phase_ms, "host": host_desc(),
                                       "observer": "digests only (≈ 1% overhead)"}).encode(), np.uint8))
    print(json.dumps({"config": a.config, "seconds": round(total, 1), "levels": len(st.levels),
                      "parts": part.num_parts, "connectivity": st.connectivity_trace[-1][-1]}))


if __name__ == "__main__":
    main()
