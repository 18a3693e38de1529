"""Generates the golden fixtures in tests/golden/ by running the REFERENCE
implementation (oracle/_ref, built from /root/reference by
oracle/build_ref.py).  Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Fixtures (small, committed):
  partition_small.npz  — 40 seeded instances: inputs + reference partition()
                         outputs (assign, num_parts, levels, trace) and the
                         per-level / per-round observer payloads
  kernels.npz          — kernel-level inputs/outputs of the reference's eight
                         dhgpart.kernels functions on seeded instances
  c1.npz               — C1 (gen 10k/20k, Omega 256, Delta 1024): assign,
                         levels, trace
  snn.npz              — a layered-SNN shape (3 x 300, Omega 64)
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref_loader  # noqa: E402
from paper_2604_14411_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent


def ref_graph(dp, arr):
    n, w, so, sd, do, dd = arr
    return dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))


def pack_run(dp, arr, omega, delta, prefix, out, record=True, max_levels=1 << 20):
    n, w, so, sd, do, dd = arr
    g = ref_graph(dp, arr)
    ev = {"level": [], "round": []}

    def obs(kind, p):
        if kind == "level":
            f = p["forest"]
            ev["level"].append((f.pair, f.score, f.match, p["cmap"].gamma, p["coarse"].edge_src.offsets,
                                p["coarse"].edge_src.data, p["coarse"].edge_dst.offsets, p["coarse"].edge_dst.data,
                                p["coarse"].node_size))
        else:
            m, s = p["moves"], p["selection"]
            ev["round"].append((p["level"], p["round"], p["assign"], m.node, m.from_part, m.to_part, m.gain_iso,
                                m.gain_seq, s.k, s.total_gain, s.active))

    part, st = dp.partition(g, dp.Config(dp.Constraints(omega, delta), max_levels=max_levels),
                            observer=obs if record else None)
    for k, v in zip(("n", "w", "so", "sd", "do", "dd"), arr):
        out[f"{prefix}in_{k}"] = np.asarray(v)
    out[f"{prefix}omega"] = np.int64(omega)
    out[f"{prefix}delta"] = np.int64(delta)
    out[f"{prefix}assign"] = part.assign
    out[f"{prefix}num_parts"] = np.int64(part.num_parts)
    out[f"{prefix}stats"] = np.frombuffer(json.dumps({"levels": st.levels, "trace": st.connectivity_trace})
                                          .encode(), dtype=np.uint8)
    if record:
        for i, t in enumerate(ev["level"]):
            for key, v in zip(("pair", "score", "match", "gamma", "so", "sd", "do", "dd", "size"), t):
                out[f"{prefix}L{i}_{key}"] = np.asarray(v)
        for i, t in enumerate(ev["round"]):
            for key, v in zip(("level", "round", "assign", "node", "from", "to", "giso", "gseq", "k", "total",
                               "active"), t):
                out[f"{prefix}R{i}_{key}"] = np.asarray(v)
        out[f"{prefix}nlev_ev"] = np.int64(len(ev["level"]))
        out[f"{prefix}nround_ev"] = np.int64(len(ev["round"]))


def partition_small(dp):
    out = {}
    rs = np.random.RandomState(2604)
    cases = []
    for t in range(40):
        n = int(rs.randint(5, 300))
        omega = int(rs.choice([2, 4, 8, 16, 32]))
        arr = W.random_dhg(n, int(1.5 * n), int(rs.choice([2, 3, 4, 5, 6])), seed=3000 + t)
        indeg = int(np.bincount(arr[5], minlength=n).max()) if len(arr[5]) else 0
        delta = max(indeg, 1) + int(rs.randint(0, 2 * omega))
        pack_run(dp, arr, omega, delta, f"c{t}_", out)
        cases.append(t)
    out["cases"] = np.asarray(cases)
    np.savez_compressed(OUT / "partition_small.npz", **out)


def kernels_fixture(dp):
    from dhgpart import kernels as K

    out = {}
    rs = np.random.RandomState(5151)
    for t in range(6):
        n = int(rs.randint(10, 120))
        arr = W.random_dhg(n, int(1.5 * n), 5, seed=5000 + t)
        g = ref_graph(dp, arr)
        omega = int(rs.choice([4, 8]))
        delta = int(g.node_in.lengths().max()) + 4
        nb = dp.materialize_neighbors(g)
        hist = K.fill_histograms(g.node_inc.offsets, g.node_inc.data, g.edge_pins.offsets, g.edge_pins.data,
                                 g.edge_weight, nb.offsets, nb.data, 7)
        seg = np.repeat(np.arange(g.num_nodes, dtype=np.int64), nb.lengths())
        order = np.lexsort((-nb.data.astype(np.int64), -hist, seg)).astype(np.int64)
        pair, score = K.select_first_valid(order, nb.offsets, nb.data, hist, g.node_size, g.node_in.offsets,
                                           g.node_in.data, omega, delta)
        match = K.resolve_matching(pair, score)
        k = max(2, n // omega)
        assign = rs.randint(0, k, size=n).astype(np.int32)
        conn = K.connectivity_value(g.edge_pins.offsets, g.edge_pins.data, g.edge_weight, assign)
        pins, pins_in = K.compute_pins(g.edge_pins.offsets, g.edge_pins.data, g.edge_dst.offsets, g.edge_dst.data,
                                       assign, k)
        psz = dp.partition_sizes(g, assign, k)
        tgt, gain = K.propose_moves(g.node_inc.offsets, g.node_inc.data, g.edge_pins.offsets, g.edge_pins.data,
                                    g.edge_weight, pins, assign, psz, g.node_size, omega)
        sel = np.flatnonzero(tgt >= 0)
        order2 = np.lexsort((sel, -gain[sel]))
        node = sel[order2].astype(np.int32)
        pos = np.full(n, -1, dtype=np.int64)
        pos[node] = np.arange(len(node))
        gseq = K.sequence_gains(g.node_inc.offsets, g.node_inc.data, g.edge_pins.offsets, g.edge_pins.data,
                                g.edge_weight, pins, node, assign[node], tgt[node].astype(np.int32), gain[node], pos)
        moves = dp.MoveSet(node=node, from_part=assign[node], to_part=tgt[node].astype(np.int32),
                           gain_iso=gain[node], gain_seq=gseq)
        pinb = dp.distinct_inbound_sizes(g, assign, k)
        s = dp.build_events_and_select(g, moves, pins_in, psz, pinb, dp.Constraints(omega, delta))
        p = f"k{t}_"
        for key, v in zip(("n", "w", "so", "sd", "do", "dd"), arr):
            out[p + "in_" + key] = np.asarray(v)
        for key, v in dict(omega=omega, delta=delta, nb_off=nb.offsets, nb_dat=nb.data, hist=hist, order=order,
                           pair=pair, score=score, match=match, K=k, assign=assign, conn=conn, pins=pins,
                           pins_in=pins_in, psz=psz, target=tgt, gain=gain, node=node, pos=pos, gseq=gseq,
                           pinb=pinb, sel_k=s.k, sel_total=s.total_gain, sel_active=s.active,
                           inc_off=g.node_inc.offsets, inc_dat=g.node_inc.data, pin_off=g.edge_pins.offsets,
                           pin_dat=g.edge_pins.data, in_off=g.node_in.offsets, in_dat=g.node_in.data,
                           out_off=g.node_out.offsets, out_dat=g.node_out.data).items():
            out[p + key] = np.asarray(v)
    out["count"] = np.int64(6)
    np.savez_compressed(OUT / "kernels.npz", **out)


def fractional(dp):
    """weights.npz: instances with fractional weights — dyadic (0.5 / 0.25
    steps: exact-integer after scaling) and decimal (0.1 steps: every f64 sum
    rounds, so only the reference's own summation order reproduces it) —
    with the reference's partition() outputs and every observer payload."""
    out = {}
    rs = np.random.RandomState(4242)
    kinds = []
    for t in range(12):
        n = int(rs.randint(30, 400))
        omega = int(rs.choice([4, 8, 16]))
        n_, w, so, sd, do, dd = W.random_dhg(n, int(1.5 * n), int(rs.choice([3, 4, 6])), seed=7000 + t)
        kind = ("half", "quarter", "decimal")[t % 3]
        if kind == "half":
            w = rs.randint(1, 20, size=len(w)) / 2.0
        elif kind == "quarter":
            w = rs.randint(1, 40, size=len(w)) / 4.0
        else:
            w = rs.randint(1, 90, size=len(w)) * 0.1
        arr = (n_, w, so, sd, do, dd)
        indeg = int(np.bincount(dd, minlength=n).max()) if len(dd) else 0
        delta = max(indeg, 1) + int(rs.randint(0, 2 * omega))
        pack_run(dp, arr, omega, delta, f"c{t}_", out)
        kinds.append(kind)
    out["kinds"] = np.asarray(kinds)
    out["cases"] = np.arange(len(kinds))
    np.savez_compressed(OUT / "weights.npz", **out)


def main():
    dp = ref_loader.load()
    if "--only" in sys.argv:
        {"fractional": fractional}[sys.argv[sys.argv.index("--only") + 1]](dp)
        return
    partition_small(dp)
    kernels_fixture(dp)
    out = {}
    pack_run(dp, W.random_dhg(10_000, 20_000, 8, seed=0), 256, 1024, "", out, record=False)
    np.savez_compressed(OUT / "c1.npz", **{k: v for k, v in out.items() if not k.startswith("in_")})
    out = {}
    pack_run(dp, W.layered_snn(3, 300), 64, 4096, "", out, record=False)
    np.savez_compressed(OUT / "snn.npz", **{k: v for k, v in out.items() if not k.startswith("in_")})
    # the reference's own generator text for a few seeds (workloads.random_dhg parity)
    texts = {f"gen_{s}": np.frombuffer(dp.generate_dhg(60, 80, 5, seed=s).encode(), dtype=np.uint8)
             for s in range(3)}
    np.savez_compressed(OUT / "gen.npz", **texts)
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
