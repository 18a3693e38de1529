"""Stepwise parity at full size: the CPU oracle cannot run
C2-C5 end to end, but level l+1 depends only on level l, and a refinement
level only on (level graph, entry assignment).  So one GPU run records the
level graphs and payloads of a few sampled levels, and the oracle replays
exactly those levels:

* coarsening: oracle.coarsen_level(graph_l) must reproduce the GPU's level-l
  event (pair, score, match, gamma and the coarse graph) bit for bit;
* refinement: oracle.refine_level(graph_l, entry assignment) must reproduce
  every round event of level l (moves, gain_iso, gain_seq, active, k) and the
  level's connectivity trace.

    python tests/stepwise_parity.py C3 --coarsen 600,1000 --refine 0,700 [--json out.json]

Test infrastructure: imports the oracle; the product never does.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time
from collections import defaultdict
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def gpu_run_sampled(g, omega, delta, coarsen_levels, refine_levels, max_rounds=8):
    """One GPU partition through dhgp_partition with an observer that keeps
    only what the sampled levels need."""
    import paper_2604_14411_b200 as dp
    from paper_2604_14411_b200 import _lib
    from paper_2604_14411_b200.driver import _make_config, _stats_from

    L = _lib.load()
    cfg = dp.Config(dp.Constraints(omega, delta), max_rounds=max_rounds, max_levels=1 << 20)
    gg, keep = g._c_graph()
    cc = _make_config(cfg)
    need = set(coarsen_levels) | set(refine_levels)
    graphs = {}
    if 0 in need:
        graphs[0] = (g.num_nodes, g.edge_src.offsets, g.edge_src.data, g.edge_dst.offsets, g.edge_dst.data,
                     np.asarray(g.node_size, dtype=np.int32))
    level_ev = {}
    rounds = defaultdict(list)
    err = []

    def cb(evp, _user):
        try:
            ev = evp.contents
            take = _lib.take
            if ev.kind == 1:
                lv, n, nc, E = ev.level, ev.num_nodes, ev.num_coarse, ev.num_edges
                if lv + 1 in need or lv in coarsen_levels:
                    so = take(ev.c_src_off, E + 1, np.int64)
                    do = take(ev.c_dst_off, E + 1, np.int64)
                    coarse = (nc, so, take(ev.c_src_dat, int(so[-1]), np.int32), do,
                              take(ev.c_dst_dat, int(do[-1]), np.int32), take(ev.c_node_size, nc, np.int32))
                    if lv + 1 in need:
                        graphs[lv + 1] = coarse
                    if lv in coarsen_levels:
                        level_ev[lv] = {"pair": take(ev.pair, n, np.int32), "score": take(ev.score, n, np.float64),
                                        "match": take(ev.match, n, np.int32), "gamma": take(ev.gamma, n, np.int32),
                                        "coarse": coarse}
            elif ev.level in refine_levels:
                m = ev.num_moves
                rounds[ev.level].append({
                    "assign": take(ev.assign, ev.num_nodes, np.int32), "num_parts": ev.num_parts,
                    "node": take(ev.mv_node, m, np.int32), "from_part": take(ev.mv_from, m, np.int32),
                    "to_part": take(ev.mv_to, m, np.int32), "gain_iso": take(ev.mv_gain_iso, m, np.float64),
                    "gain_seq": take(ev.mv_gain_seq, m, np.float64), "k": ev.k, "total_gain": ev.total_gain,
                    "active": take(ev.active, m + 1, np.int64)})
        except BaseException as ex:  # re-raised below
            err.append(ex)

    ocb = _lib.OBSERVER(cb)
    assign = np.zeros(max(g.num_nodes, 1), dtype=np.int32)
    nparts = C.c_int32(0)
    st = _lib.DhgpStats()
    rc = L.dhgp_partition(C.byref(gg), C.byref(cc), _lib.ptr(assign), C.byref(nparts), C.byref(st), ocb, None)
    del keep
    if err:
        raise err[0]
    _lib.raise_for(rc)
    stats = _stats_from(L, st, False)
    return stats, graphs, level_ev, rounds


_JOBS: list = []  # (kind, level, args) set before the pool forks; workers get an index


def _replay(i):
    from oracle import oracle as orc

    kind, lv, args, kw = _JOBS[i]
    t = time.time()
    out = orc.coarsen_level(*args, **kw) if kind == "c" else orc.refine_level(*args, **kw)
    return i, out, time.time() - t


def auto_levels(nlev: int):
    """Early levels (where the full / block / dense scoring tiers run on the
    most nodes) plus levels spread to the tail."""
    co = {0, 1, 2, 8, 32} | {int(round(x)) for x in np.linspace(64, nlev - 2, 6)}
    re = {0, 1, nlev // 2, nlev - 2, nlev - 1}
    return sorted(x for x in co if 0 <= x < nlev - 1), sorted(x for x in re if 0 <= x < nlev)


def check_config(name, coarsen_levels, refine_levels, log=print, procs=None):
    import multiprocessing as mp

    import paper_2604_14411_b200 as dp
    from paper_2604_14411_b200 import workloads as W

    arrs, omega, delta, desc = W.make_config(name)
    n, w, so, sd, do, dd = arrs
    g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
    if coarsen_levels is None or refine_levels is None:  # auto: needs the level count first
        _, st0 = dp.partition(g, dp.Config(dp.Constraints(omega, delta), max_levels=1 << 20))
        ac, ar = auto_levels(len(st0.levels))
        coarsen_levels = ac if coarsen_levels is None else coarsen_levels
        refine_levels = ar if refine_levels is None else refine_levels
    t0 = time.time()
    stats, graphs, level_ev, rounds = gpu_run_sampled(g, omega, delta, coarsen_levels, refine_levels)
    nlev = len(stats.levels)
    out = {"config": name, "desc": desc, "levels": nlev, "gpu_run_s": round(time.time() - t0, 2),
           "coarsen": [], "refine": []}
    _JOBS.clear()
    for lv in sorted(coarsen_levels):
        if lv < nlev - 1:
            gl = graphs[lv]
            _JOBS.append(("c", lv, (gl[0], w, gl[1], gl[2], gl[3], gl[4], gl[5]),
                          dict(max_size=omega, max_inbound=delta)))
    for lv in sorted(refine_levels):
        if lv < nlev and rounds.get(lv):
            gl = graphs[lv]
            _JOBS.append(("r", lv, (gl[0], w, gl[1], gl[2], gl[3], gl[4], gl[5], rounds[lv][0]["assign"],
                                    rounds[lv][0]["num_parts"]), dict(max_size=omega, max_inbound=delta, level=lv)))
    procs = procs or max(1, min(len(_JOBS), (os.cpu_count() or 2) - 1))
    results = {}
    # largest levels first so the pool's tail is short
    order = sorted(range(len(_JOBS)), key=lambda i: -len(_JOBS[i][2][2]) - len(_JOBS[i][2][4]))
    with mp.get_context("fork").Pool(procs) as pool:
        for i, res, secs in pool.imap_unordered(_replay, order):
            results[i] = (res, secs)
    for i, (kind, lv, args, _) in enumerate(_JOBS):
        ref, secs = results[i]
        gl = graphs[lv]
        if kind == "c":
            mine = level_ev[lv]
            ok = ref is not None and all(np.array_equal(ref[k], mine[k]) for k in ("pair", "score", "match", "gamma"))
            c = mine["coarse"]
            ok = ok and ref["num_coarse"] == c[0] and all(
                np.array_equal(ref[k], v)
                for k, v in zip(("src_off", "src_dat", "dst_off", "dst_dat", "node_size"), c[1:]))
            rec = {"level": lv, "nodes": int(gl[0]), "pins": int(len(gl[2]) + len(gl[4])),
                   "coarse_nodes": int(c[0]), "pairs": int(np.sum(mine["match"] != np.arange(gl[0])) // 2),
                   "bit_exact": bool(ok), "oracle_s": round(secs, 2)}
            if not ok and ref is not None:  # diagnostics: which payload differs, and where first
                diff = {}
                for k in ("pair", "score", "match", "gamma"):
                    a_, b_ = np.asarray(ref[k]), np.asarray(mine[k])
                    if a_.shape != b_.shape:
                        diff[k] = f"shape {a_.shape} vs {b_.shape}"
                    elif not np.array_equal(a_, b_):
                        bad = np.flatnonzero(a_ != b_)
                        i0 = int(bad[0])
                        diff[k] = {"count": int(len(bad)), "first": i0, "oracle": a_[i0].item(),
                                   "gpu": b_[i0].item()}
                        if k == "pair":
                            diff[k]["score_oracle"] = float(ref["score"][i0])
                            diff[k]["score_gpu"] = float(mine["score"][i0])
                if ref["num_coarse"] != c[0]:
                    diff["num_coarse"] = [int(ref["num_coarse"]), int(c[0])]
                for k, v in zip(("src_off", "src_dat", "dst_off", "dst_dat", "node_size"), c[1:]):
                    a_, b_ = np.asarray(ref[k]), np.asarray(v)
                    if a_.shape != b_.shape:
                        diff[k] = f"shape {a_.shape} vs {b_.shape}"
                    elif not np.array_equal(a_, b_):
                        bad = np.flatnonzero(a_ != b_)
                        i0 = int(bad[0])
                        diff[k] = {"count": int(len(bad)), "first": i0, "oracle": a_[max(0, i0 - 3):i0 + 4].tolist(),
                                   "gpu": b_[max(0, i0 - 3):i0 + 4].tolist()}
                        if k.endswith("_dat"):  # the owning h-edge and its lists
                            off_o = np.asarray(ref[k[:3] + "_off"])
                            e = int(np.searchsorted(off_o, i0, side="right") - 1)
                            off_g = np.asarray(c[1] if k == "src_dat" else c[3])
                            diff[k]["edge"] = e
                            diff[k]["edge_oracle"] = a_[off_o[e]:off_o[e + 1]].tolist()
                            diff[k]["edge_gpu"] = b_[off_g[e]:off_g[e + 1]].tolist()
                            fo, fd = (gl[1], gl[2]) if k == "src_dat" else (gl[3], gl[4])
                            diff[k]["edge_fine"] = np.asarray(fd[fo[e]:fo[e + 1]]).tolist()
                rec["diff"] = diff
            out["coarsen"].append(rec)
        else:
            a, conns, evs = ref
            rs = rounds[lv]
            ok = len(evs) == len(rs)
            for e, r in zip(evs, rs):
                ok = ok and e["k"] == r["k"] and e["total_gain"] == r["total_gain"] and all(
                    np.array_equal(e[k], r[k]) for k in ("assign", "node", "from_part", "to_part", "gain_iso",
                                                         "gain_seq", "active"))
            ok = ok and conns == stats.connectivity_trace[nlev - 1 - lv]
            rec = {"level": lv, "nodes": int(gl[0]), "rounds": len(rs),
                   "moves": int(sum(len(r["node"]) for r in rs)), "bit_exact": bool(ok), "oracle_s": round(secs, 2)}
            out["refine"].append(rec)
        log(json.dumps(rec))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--coarsen", default="auto", help="comma list of levels, or 'auto'")
    ap.add_argument("--refine", default="auto", help="comma list of levels, or 'auto'")
    ap.add_argument("--head", default=None, help="commit the product code was built from (recorded)")
    ap.add_argument("--procs", type=int, default=None, help="oracle replays in parallel (fork)")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    lv = lambda s: None if s == "auto" else [int(x) for x in s.split(",") if x != ""]  # noqa: E731
    out = check_config(a.config, lv(a.coarsen), lv(a.refine), procs=a.procs)
    out["head"] = a.head
    print(json.dumps({k: v for k, v in out.items() if k not in ("coarsen", "refine")}))
    if a.json:
        Path(a.json).write_text(json.dumps(out, indent=1))
    ok = all(r["bit_exact"] for r in out["coarsen"] + out["refine"])
    print("STEPWISE", "OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
