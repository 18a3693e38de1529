"""Diagnostic: GPU partition vs oracle with per-level / per-round diffs.

Run on a GPU box:  python tests/diag_parity.py [--big]
Prints the first differing level or round for any mismatching instance.
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2604_14411_b200 as dp  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2604_14411_b200 import workloads as W  # noqa: E402


def gpu_run(arr, omega, delta, **kw):
    n, w, so, sd, do, dd = arr
    g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
    events = []

    def obs(kind, p):
        if kind == "level":
            events.append({"kind": "level", "index": p["index"], "pair": p["forest"].pair,
                           "score": p["forest"].score, "match": p["forest"].match, "gamma": p["cmap"].gamma,
                           "src_off": p["coarse"].edge_src.offsets, "src_dat": p["coarse"].edge_src.data,
                           "dst_off": p["coarse"].edge_dst.offsets, "dst_dat": p["coarse"].edge_dst.data,
                           "node_size": p["coarse"].node_size})
        else:
            m = p["moves"]
            events.append({"kind": "round", "level": p["level"], "round": p["round"], "assign": p["assign"],
                           "node": m.node, "from_part": m.from_part, "to_part": m.to_part, "gain_iso": m.gain_iso,
                           "gain_seq": m.gain_seq, "k": p["selection"].k, "total_gain": p["selection"].total_gain,
                           "active": p["selection"].active})

    t = time.perf_counter()
    part, stats = dp.partition(g, dp.Config(dp.Constraints(omega, delta), **kw), observer=obs if kw.pop("_obs", True) else None)
    return part, stats, events, time.perf_counter() - t


def compare(arr, omega, delta, label, max_levels=1 << 20, observe=True):
    n, w, so, sd, do, dd = arr
    try:
        a, k, st, oev = orc.partition(n, w, so, sd, do, dd, max_size=omega, max_inbound=delta,
                                      max_levels=max_levels, record=observe)
    except orc.OracleError as ex:
        oev = None
        ref_err = ex
    else:
        ref_err = None
    try:
        if observe:
            part, stats, gev, dt = gpu_run(arr, omega, delta, max_levels=max_levels)
        else:
            g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
            t = time.perf_counter()
            part, stats = dp.partition(g, dp.Config(dp.Constraints(omega, delta), max_levels=max_levels))
            dt = time.perf_counter() - t
            gev = []
    except dp.DhgError as ex:
        if ref_err is not None:
            print(f"{label}: both raised ({type(ex).__name__} / code {ref_err.code})")
            return True
        print(f"{label}: GPU raised {type(ex).__name__}: {ex}")
        return False
    if ref_err is not None:
        print(f"{label}: oracle raised {ref_err} but GPU did not")
        return False
    ok = (np.array_equal(part.assign, a) and part.num_parts == k and stats.levels == st["levels"]
          and stats.connectivity_trace == st["connectivity_trace"])
    if ok:
        print(f"{label}: OK  levels={len(stats.levels)} parts={k} conn={st['connectivity_trace'][-1][-1]} "
              f"gpu={dt*1e3:.1f} ms launches={stats._gpu_launches}")
        return True
    print(f"{label}: MISMATCH levels gpu={len(stats.levels)} ref={len(st['levels'])}")
    for i, (ge, oe) in enumerate(zip(gev, oev)):
        if ge["kind"] != oe["kind"]:
            print(f"  event {i}: kind {ge['kind']} vs {oe['kind']}")
            return False
        for key in ge:
            if key == "kind":
                continue
            gv, ov = ge[key], oe.get(key)
            same = np.array_equal(np.asarray(gv), np.asarray(ov)) if isinstance(gv, np.ndarray) else gv == ov
            if not same:
                print(f"  event {i} ({ge['kind']} level={ge.get('index', ge.get('level'))} "
                      f"round={ge.get('round')}): field {key} differs")
                gv, ov = np.asarray(gv), np.asarray(ov)
                if gv.shape == ov.shape and gv.ndim == 1:
                    bad = np.flatnonzero(gv != ov)
                    print(f"    first diffs at {bad[:10].tolist()}: gpu {gv[bad[:10]].tolist()} "
                          f"ref {ov[bad[:10]].tolist()}")
                else:
                    print(f"    gpu {gv[:20]} ... ref {ov[:20]}")
                return False
    print(f"  events equal for {min(len(gev), len(oev))} events; counts gpu={len(gev)} ref={len(oev)}")
    return False


def main():
    big = "--big" in sys.argv
    ok = True
    ok &= compare(W.random_dhg(4, 3, 2, seed=1), 2, 4, "tiny")
    rs = np.random.RandomState(3)
    for t in range(40):
        n = int(rs.randint(5, 500))
        omega = int(rs.choice([2, 4, 8, 16, 32]))
        arr = W.random_dhg(n, int(1.5 * n), int(rs.choice([2, 3, 4, 5, 6])), seed=100 + t)
        indeg = np.bincount(arr[5], minlength=n).max()
        ok &= compare(arr, omega, int(max(indeg, 1) + rs.randint(0, 2 * omega)), f"rand{t}")
    ok &= compare(W.layered_snn(3, 300), 64, 4096, "snn3x300")
    ok &= compare(W.random_dhg(10000, 20000, 8, seed=0), 256, 1024, "C1", observe=False)
    if big:
        ok &= compare(W.layered_snn(4, 400), 128, 4096, "snn4x400")
        ok &= compare(W.layered_snn(5, 1000), 1024, 4096, "snn5x1000", observe=False)
    print("ALL OK" if ok else "FAILURES")


if __name__ == "__main__":
    main()
