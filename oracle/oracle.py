"""ctypes wrapper around oracle/liboracle.so — TEST INFRASTRUCTURE ONLY.

The oracle is a sequential C restatement of the reference partitioner
(see dhgp_oracle.c).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
I64P = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class DhgpEvent(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("level", C.c_int32), ("round", C.c_int32),
        ("num_nodes", C.c_int32), ("num_edges", C.c_int32), ("num_coarse", C.c_int32),
        ("num_parts", C.c_int32),
        ("pair", C.POINTER(C.c_int32)), ("score", C.POINTER(C.c_double)),
        ("match", C.POINTER(C.c_int32)), ("gamma", C.POINTER(C.c_int32)),
        ("c_src_off", C.POINTER(C.c_int64)), ("c_src_dat", C.POINTER(C.c_int32)),
        ("c_dst_off", C.POINTER(C.c_int64)), ("c_dst_dat", C.POINTER(C.c_int32)),
        ("c_node_size", C.POINTER(C.c_int32)),
        ("assign", C.POINTER(C.c_int32)), ("num_moves", C.c_int32),
        ("mv_node", C.POINTER(C.c_int32)), ("mv_from", C.POINTER(C.c_int32)),
        ("mv_to", C.POINTER(C.c_int32)), ("mv_gain_iso", C.POINTER(C.c_double)),
        ("mv_gain_seq", C.POINTER(C.c_double)), ("k", C.c_int32),
        ("total_gain", C.c_double), ("active", C.POINTER(C.c_int64)),
    ]


class DhgpStats(C.Structure):
    _fields_ = [
        ("num_levels", C.c_int64),
        ("level_nodes", C.POINTER(C.c_int64)), ("level_edges", C.POINTER(C.c_int64)),
        ("level_pins", C.POINTER(C.c_int64)),
        ("trace_off", C.POINTER(C.c_int64)), ("trace_val", C.POINTER(C.c_double)),
        ("num_partitions", C.c_int32), ("phase_ms", C.c_double * 3),
        ("gpu_launches", C.c_int64), ("device_ms", C.c_double),
    ]


OBSERVER = C.CFUNCTYPE(None, C.POINTER(DhgpEvent), C.c_void_p)


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build(force: bool = False) -> Path:
    src = HERE / "dhgp_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-o", str(LIB_PATH), str(src)], cwd=str(HERE)
        )
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.orc_last_error.restype = C.c_char_p
        L.orc_connectivity_value.restype = C.c_double
        L.orc_union_size_sorted.restype = C.c_int64
        L.orc_build_events_and_select.restype = C.c_int64
        L.orc_neighbors_count.restype = C.c_int64
        _lib = L
    return _lib


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def event_to_dict(ev: DhgpEvent) -> dict:
    """Copy one observer event into plain numpy arrays."""
    if ev.kind == 1:
        n, nc, E = ev.num_nodes, ev.num_coarse, ev.num_edges
        src_off = _arr(ev.c_src_off, E + 1, np.int64)
        dst_off = _arr(ev.c_dst_off, E + 1, np.int64)
        return {
            "kind": "level", "index": ev.level, "num_nodes": n, "num_coarse": nc,
            "pair": _arr(ev.pair, n, np.int32), "score": _arr(ev.score, n, np.float64),
            "match": _arr(ev.match, n, np.int32), "gamma": _arr(ev.gamma, n, np.int32),
            "src_off": src_off, "src_dat": _arr(ev.c_src_dat, int(src_off[-1]), np.int32),
            "dst_off": dst_off, "dst_dat": _arr(ev.c_dst_dat, int(dst_off[-1]), np.int32),
            "node_size": _arr(ev.c_node_size, nc, np.int32),
        }
    m = ev.num_moves
    return {
        "kind": "round", "level": ev.level, "round": ev.round, "num_parts": ev.num_parts,
        "assign": _arr(ev.assign, ev.num_nodes, np.int32),
        "node": _arr(ev.mv_node, m, np.int32), "from_part": _arr(ev.mv_from, m, np.int32),
        "to_part": _arr(ev.mv_to, m, np.int32), "gain_iso": _arr(ev.mv_gain_iso, m, np.float64),
        "gain_seq": _arr(ev.mv_gain_seq, m, np.float64), "k": ev.k,
        "total_gain": ev.total_gain, "active": _arr(ev.active, m + 1, np.int64),
    }


def partition(num_nodes, weights, src_off, src_dat, dst_off, dst_dat, node_size=None, *,
              max_size, max_inbound, max_rounds=8, max_levels=64, record=False):
    """Full pipeline.  Returns (assign, num_parts, stats_dict, events)."""
    L = lib()
    w = _c(weights, np.float64)
    E = len(w)
    so, sd = _c(src_off, np.int64), _c(src_dat, np.int32)
    do, dd = _c(dst_off, np.int64), _c(dst_dat, np.int32)
    ns = None if node_size is None else _c(node_size, np.int32)
    assign = np.zeros(max(num_nodes, 1), dtype=np.int32)
    nparts = C.c_int32(0)
    st = DhgpStats()
    events: list[dict] = []

    def _obs(evp, _user):
        events.append(event_to_dict(evp.contents))

    cb = OBSERVER(_obs) if record else OBSERVER()
    rc = L.orc_partition(
        C.c_int32(num_nodes), C.c_int32(E), w.ctypes.data_as(C.c_void_p),
        so.ctypes.data_as(C.c_void_p), sd.ctypes.data_as(C.c_void_p),
        do.ctypes.data_as(C.c_void_p), dd.ctypes.data_as(C.c_void_p),
        None if ns is None else ns.ctypes.data_as(C.c_void_p),
        C.c_int64(max_size), C.c_int64(max_inbound), C.c_int32(max_rounds), C.c_int32(max_levels),
        assign.ctypes.data_as(C.c_void_p), C.byref(nparts), C.byref(st), cb, None,
    )
    if rc != 0:
        raise OracleError(rc, L.orc_last_error().decode())
    nl = st.num_levels
    tro = _arr(st.trace_off, nl + 1, np.int64)
    trv = _arr(st.trace_val, int(tro[-1]), np.float64)
    stats = {
        "levels": [
            {"nodes": int(st.level_nodes[i]), "edges": int(st.level_edges[i]), "pins": int(st.level_pins[i])}
            for i in range(nl)
        ],
        "connectivity_trace": [trv[tro[i]:tro[i + 1]].tolist() for i in range(nl)],
        "num_partitions": int(st.num_partitions),
    }
    L.orc_stats_free(C.byref(st))
    return assign[:num_nodes].copy(), int(nparts.value), stats, events


# ---- kernel-level mirrors (same argument meaning as dhgpart.kernels) ----

def incidence(num_nodes, src_off, src_dat, dst_off, dst_dat):
    L = lib()
    so, sd = _c(src_off, np.int64), _c(src_dat, np.int32)
    do, dd = _c(dst_off, np.int64), _c(dst_dat, np.int32)
    E = len(so) - 1
    N = num_nodes
    cap = int(so[-1] - so[0] + do[-1] - do[0])
    in_off = np.zeros(N + 1, np.int64); in_dat = np.zeros(max(int(do[-1] - do[0]), 1), np.int32)
    out_off = np.zeros(N + 1, np.int64); out_dat = np.zeros(max(int(so[-1] - so[0]), 1), np.int32)
    pin_off = np.zeros(E + 1, np.int64); pin_dat = np.zeros(max(cap, 1), np.int32)
    inc_off = np.zeros(N + 1, np.int64); inc_dat = np.zeros(max(cap, 1), np.int32)
    L.orc_incidence(C.c_int32(N), C.c_int32(E), *(a.ctypes.data_as(C.c_void_p) for a in (
        so, sd, do, dd, in_off, in_dat, out_off, out_dat, pin_off, pin_dat, inc_off, inc_dat)))
    return {
        "node_in": (in_off, in_dat[: in_off[-1]]), "node_out": (out_off, out_dat[: out_off[-1]]),
        "edge_pins": (pin_off, pin_dat[: pin_off[-1]]), "node_inc": (inc_off, inc_dat[: inc_off[-1]]),
    }


def neighbors(num_nodes, src_off, src_dat, dst_off, dst_dat):
    L = lib()
    so, sd = _c(src_off, np.int64), _c(src_dat, np.int32)
    do, dd = _c(dst_off, np.int64), _c(dst_dat, np.int32)
    E = len(so) - 1
    args = (C.c_int32(num_nodes), C.c_int32(E), *(a.ctypes.data_as(C.c_void_p) for a in (so, sd, do, dd)))
    nnz = L.orc_neighbors_count(*args)
    off = np.zeros(num_nodes + 1, np.int64)
    dat = np.zeros(max(nnz, 1), np.int32)
    L.orc_neighbors(*args, off.ctypes.data_as(C.c_void_p), dat.ctypes.data_as(C.c_void_p))
    return off, dat[:nnz]


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def fill_histograms(inc_off, inc_dat, pin_off, pin_dat, w, nbr_off, nbr_dat):
    inc_off, inc_dat = _c(inc_off, np.int64), _c(inc_dat, np.int32)
    pin_off, pin_dat = _c(pin_off, np.int64), _c(pin_dat, np.int32)
    w, nbr_off, nbr_dat = _c(w, np.float64), _c(nbr_off, np.int64), _c(nbr_dat, np.int32)
    hist = np.zeros(max(len(nbr_dat), 1), np.float64)
    lib().orc_fill_histograms(C.c_int32(len(nbr_off) - 1), _p(inc_off), _p(inc_dat), _p(pin_off), _p(pin_dat),
                              _p(w), _p(nbr_off), _p(nbr_dat), _p(hist))
    return hist[: len(nbr_dat)]


def select_first_valid(nbr_off, nbr_dat, hist, node_size, in_off, in_dat, max_size, max_inbound):
    nbr_off, nbr_dat, hist = _c(nbr_off, np.int64), _c(nbr_dat, np.int32), _c(hist, np.float64)
    node_size, in_off, in_dat = _c(node_size, np.int32), _c(in_off, np.int64), _c(in_dat, np.int32)
    n = len(nbr_off) - 1
    pair = np.zeros(max(n, 1), np.int32)
    score = np.zeros(max(n, 1), np.float64)
    lib().orc_select_first_valid(C.c_int32(n), _p(nbr_off), _p(nbr_dat), _p(hist), _p(node_size), _p(in_off),
                                 _p(in_dat), C.c_int64(max_size), C.c_int64(max_inbound), _p(pair), _p(score))
    return pair[:n], score[:n]


def resolve_matching(pair, score):
    pair, score = _c(pair, np.int32), _c(score, np.float64)
    n = len(pair)
    match = np.zeros(max(n, 1), np.int32)
    rc = lib().orc_resolve_matching(C.c_int32(n), _p(pair), _p(score), _p(match))
    if rc:
        raise OracleError(rc, lib().orc_last_error().decode())
    return match[:n]


def connectivity_value(pin_off, pin_dat, w, assign):
    pin_off, pin_dat, w, assign = _c(pin_off, np.int64), _c(pin_dat, np.int32), _c(w, np.float64), _c(assign, np.int32)
    return float(lib().orc_connectivity_value(C.c_int32(len(w)), _p(pin_off), _p(pin_dat), _p(w), _p(assign)))


def compute_pins(pin_off, pin_dat, dst_off, dst_dat, assign, num_parts):
    pin_off, pin_dat = _c(pin_off, np.int64), _c(pin_dat, np.int32)
    dst_off, dst_dat, assign = _c(dst_off, np.int64), _c(dst_dat, np.int32), _c(assign, np.int32)
    E = len(pin_off) - 1
    pins = np.zeros((E, num_parts), np.int32)
    pins_in = np.zeros((E, num_parts), np.int32)
    lib().orc_compute_pins(C.c_int32(E), _p(pin_off), _p(pin_dat), _p(dst_off), _p(dst_dat), _p(assign),
                           C.c_int32(num_parts), _p(pins), _p(pins_in))
    return pins, pins_in


def propose_moves(inc_off, inc_dat, pin_off, pin_dat, w, pins, assign, part_sizes, node_size, max_size):
    inc_off, inc_dat = _c(inc_off, np.int64), _c(inc_dat, np.int32)
    pin_off, pin_dat, w = _c(pin_off, np.int64), _c(pin_dat, np.int32), _c(w, np.float64)
    pins, assign = _c(pins, np.int32), _c(assign, np.int32)
    part_sizes, node_size = _c(part_sizes, np.int64), _c(node_size, np.int32)
    n = len(inc_off) - 1
    K = pins.shape[1] if pins.ndim == 2 else 0
    target = np.zeros(max(n, 1), np.int32)
    gain = np.zeros(max(n, 1), np.float64)
    lib().orc_propose_moves(C.c_int32(n), C.c_int32(K), _p(inc_off), _p(inc_dat), _p(pin_off), _p(pin_dat), _p(w),
                            _p(pins), _p(assign), _p(part_sizes), _p(node_size), C.c_int64(max_size), _p(target),
                            _p(gain))
    return target[:n], gain[:n]


def sequence_gains(inc_off, inc_dat, pin_off, pin_dat, w, pins, node, from_part, to_part, gain_iso, pos):
    inc_off, inc_dat = _c(inc_off, np.int64), _c(inc_dat, np.int32)
    pin_off, pin_dat, w = _c(pin_off, np.int64), _c(pin_dat, np.int32), _c(w, np.float64)
    pins = _c(pins, np.int32)
    node, from_part, to_part = _c(node, np.int32), _c(from_part, np.int32), _c(to_part, np.int32)
    gain_iso, pos = _c(gain_iso, np.float64), _c(pos, np.int64)
    m = len(node)
    out = np.zeros(max(m, 1), np.float64)
    lib().orc_sequence_gains(C.c_int32(m), C.c_int32(pins.shape[1]), _p(inc_off), _p(inc_dat), _p(pin_off),
                             _p(pin_dat), _p(w), _p(pins), _p(node), _p(from_part), _p(to_part), _p(gain_iso),
                             _p(pos), _p(out))
    return out[:m]


def build_events_and_select(num_nodes, num_edges, in_off, in_dat, node_size, node, from_part, to_part, gain_seq,
                            pins_in, part_sizes, part_inbound, max_size, max_inbound):
    in_off, in_dat, node_size = _c(in_off, np.int64), _c(in_dat, np.int32), _c(node_size, np.int32)
    node, from_part, to_part = _c(node, np.int32), _c(from_part, np.int32), _c(to_part, np.int32)
    gain_seq, pins_in = _c(gain_seq, np.float64), _c(pins_in, np.int32)
    part_sizes, part_inbound = _c(part_sizes, np.int64), _c(part_inbound, np.int64)
    m = len(node)
    active = np.zeros(m + 1, np.int64)
    tg = C.c_double(0.0)
    k = lib().orc_build_events_and_select(
        C.c_int32(num_nodes), C.c_int32(num_edges), _p(in_off), _p(in_dat), _p(node_size),
        C.c_int32(pins_in.shape[1]), C.c_int32(m), _p(node), _p(from_part), _p(to_part), _p(gain_seq),
        _p(pins_in), _p(part_sizes), _p(part_inbound), C.c_int64(max_size), C.c_int64(max_inbound),
        _p(active), C.byref(tg))
    return int(k), float(tg.value), active


def union_size_sorted(a, b):
    a, b = _c(a, np.int32), _c(b, np.int32)
    return int(lib().orc_union_size_sorted(_p(a), C.c_int64(len(a)), _p(b), C.c_int64(len(b))))


# ---- stepwise replay: one level of a run too large for the CPU ----

def coarsen_level(num_nodes, weights, src_off, src_dat, dst_off, dst_dat, node_size, *, max_size, max_inbound):
    """One coarsening level (coarsen.py:93-173) of the given level graph: the
    payload of its "level" event (pair, score, match, gamma, coarse graph),
    or None when the level finds no pair.  Level l+1 depends only on level l
    (the carried neighbour sets equal the rematerialised ones)."""
    L = lib()
    w = _c(weights, np.float64)
    so, sd = _c(src_off, np.int64), _c(src_dat, np.int32)
    do, dd = _c(dst_off, np.int64), _c(dst_dat, np.int32)
    ns = _c(node_size, np.int32)
    assign = np.zeros(max(num_nodes, 1), dtype=np.int32)
    nparts = C.c_int32(0)
    st = DhgpStats()
    events: list[dict] = []

    def _obs(evp, _user):
        if evp.contents.kind == 1:
            events.append(event_to_dict(evp.contents))

    cb = OBSERVER(_obs)
    L.orc_partition(
        C.c_int32(num_nodes), C.c_int32(len(w)), w.ctypes.data_as(C.c_void_p),
        so.ctypes.data_as(C.c_void_p), sd.ctypes.data_as(C.c_void_p),
        do.ctypes.data_as(C.c_void_p), dd.ctypes.data_as(C.c_void_p), ns.ctypes.data_as(C.c_void_p),
        C.c_int64(max_size), C.c_int64(max_inbound), C.c_int32(1), C.c_int32(1),
        assign.ctypes.data_as(C.c_void_p), C.byref(nparts), C.byref(st), cb, None,
    )
    L.orc_stats_free(C.byref(st))
    return events[0] if events else None


def refine_level(num_nodes, weights, src_off, src_dat, dst_off, dst_dat, node_size, assign, num_parts, *,
                 max_size, max_inbound, max_rounds=8, level=0):
    """refine_level (refine.py:262-318) of one level graph from an entry
    assignment: (final assign, connectivity trace, round events)."""
    L = lib()
    w = _c(weights, np.float64)
    so, sd = _c(src_off, np.int64), _c(src_dat, np.int32)
    do, dd = _c(dst_off, np.int64), _c(dst_dat, np.int32)
    ns = _c(node_size, np.int32)
    a = np.array(assign, dtype=np.int32, copy=True)
    conns = np.zeros(max_rounds + 1, dtype=np.float64)
    nc = C.c_int64(0)
    events: list[dict] = []

    def _obs(evp, _user):
        events.append(event_to_dict(evp.contents))

    cb = OBSERVER(_obs)
    L.orc_refine_level(
        C.c_int32(num_nodes), C.c_int32(len(w)), w.ctypes.data_as(C.c_void_p),
        so.ctypes.data_as(C.c_void_p), sd.ctypes.data_as(C.c_void_p),
        do.ctypes.data_as(C.c_void_p), dd.ctypes.data_as(C.c_void_p), ns.ctypes.data_as(C.c_void_p),
        a.ctypes.data_as(C.c_void_p), C.c_int32(num_parts), C.c_int64(max_size), C.c_int64(max_inbound),
        C.c_int32(max_rounds), C.c_int32(level), cb, None, conns.ctypes.data_as(C.c_void_p), C.byref(nc),
    )
    return a[:num_nodes], conns[: nc.value].tolist(), events
