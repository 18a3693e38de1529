"""The reference's kernel operator API (dhgpart.kernels, kernels.py:14-103),
served by one backend: libdhgp.so on the GPU.

Same eight functions, argument order, dtypes and return values; each call
is one C-ABI seam (include/dhgp.h).  There is no multi-backend dispatch:
``available_backends()`` is ``["cuda"]`` and ``set_backend`` accepts only
that name.  ``batch`` is validated and result-invariant, as in the
reference.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import DhgError

_BACKEND = "cuda"


def available_backends() -> list[str]:
    return [_BACKEND]


def active_backend() -> str:
    return _BACKEND


def set_backend(name: str) -> str:
    if name != _BACKEND:
        raise ValueError(f"unknown backend {name!r} (have: {available_backends()})")
    return _BACKEND


def get_module(name: str | None = None):
    if name not in (None, _BACKEND):
        raise ValueError(f"unknown backend {name!r} (have: {available_backends()})")
    import sys

    return sys.modules[__name__]


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _dev():
    return C.c_int32(_lib.device())


def union_size_sorted(a, b) -> int:
    a, b = _i32(a), _i32(b)
    out = C.c_int64(0)
    _lib.raise_for(_lib.load().dhgp_union_size_sorted(_lib.ptr(a), C.c_int64(len(a)), _lib.ptr(b),
                                                      C.c_int64(len(b)), _dev(), C.byref(out)))
    return int(out.value)


def fill_histograms(inc_off, inc_dat, pin_off, pin_dat, w, nbr_off, nbr_dat, batch):
    inc_off, inc_dat, pin_off, pin_dat = _i64(inc_off), _i32(inc_dat), _i64(pin_off), _i32(pin_dat)
    w, nbr_off, nbr_dat = _f64(w), _i64(nbr_off), _i32(nbr_dat)
    hist = np.zeros(max(len(nbr_dat), 1), dtype=np.float64)
    rc = _lib.load().dhgp_fill_histograms(
        C.c_int32(len(inc_off) - 1), _lib.ptr(inc_off), _lib.ptr(inc_dat), C.c_int32(len(pin_off) - 1),
        _lib.ptr(pin_off), _lib.ptr(pin_dat), _lib.ptr(w), _lib.ptr(nbr_off), _lib.ptr(nbr_dat),
        C.c_int64(int(batch)), _dev(), _lib.ptr(hist))
    _lib.raise_for(rc)
    return hist[: len(nbr_dat)]


def select_first_valid(order, nbr_off, nbr_dat, hist, node_size, in_off, in_dat, max_size, max_inbound):
    order, nbr_off, nbr_dat, hist = _i64(order), _i64(nbr_off), _i32(nbr_dat), _f64(hist)
    node_size, in_off, in_dat = _i32(node_size), _i64(in_off), _i32(in_dat)
    n = len(nbr_off) - 1
    pair = np.zeros(max(n, 1), dtype=np.int32)
    score = np.zeros(max(n, 1), dtype=np.float64)
    rc = _lib.load().dhgp_select_first_valid(
        C.c_int32(n), _lib.ptr(order), _lib.ptr(nbr_off), _lib.ptr(nbr_dat), _lib.ptr(hist), _lib.ptr(node_size),
        _lib.ptr(in_off), _lib.ptr(in_dat), C.c_int64(int(max_size)), C.c_int64(int(max_inbound)), _dev(),
        _lib.ptr(pair), _lib.ptr(score))
    _lib.raise_for(rc)
    return pair[:n], score[:n]


def resolve_matching(pair, score):
    pair, score = _i32(pair), _f64(score)
    n = len(pair)
    match = np.zeros(max(n, 1), dtype=np.int32)
    rc = _lib.load().dhgp_resolve_matching(C.c_int32(n), _lib.ptr(pair), _lib.ptr(score), _dev(), _lib.ptr(match))
    _lib.raise_for(rc)
    return match[:n]


def connectivity_value(pin_off, pin_dat, w, assign):
    pin_off, pin_dat, w, assign = _i64(pin_off), _i32(pin_dat), _f64(w), _i32(assign)
    out = C.c_double(0.0)
    rc = _lib.load().dhgp_connectivity_value(
        C.c_int32(len(w)), _lib.ptr(pin_off), _lib.ptr(pin_dat), _lib.ptr(w), C.c_int32(len(assign)),
        _lib.ptr(assign), _dev(), C.byref(out))
    _lib.raise_for(rc)
    return float(out.value)


def compute_pins(pin_off, pin_dat, dst_off, dst_dat, assign, num_parts):
    pin_off, pin_dat, dst_off, dst_dat, assign = _i64(pin_off), _i32(pin_dat), _i64(dst_off), _i32(dst_dat), _i32(assign)
    E = len(pin_off) - 1
    pins = np.zeros((E, int(num_parts)), dtype=np.int32)
    pins_in = np.zeros((E, int(num_parts)), dtype=np.int32)
    rc = _lib.load().dhgp_compute_pins(
        C.c_int32(E), _lib.ptr(pin_off), _lib.ptr(pin_dat), _lib.ptr(dst_off), _lib.ptr(dst_dat),
        C.c_int32(len(assign)), _lib.ptr(assign), C.c_int32(int(num_parts)), _dev(), _lib.ptr(pins),
        _lib.ptr(pins_in))
    _lib.raise_for(rc)
    return pins, pins_in


def propose_moves(inc_off, inc_dat, pin_off, pin_dat, w, pins, assign, part_sizes, node_size, max_size):
    inc_off, inc_dat, pin_off, pin_dat, w = _i64(inc_off), _i32(inc_dat), _i64(pin_off), _i32(pin_dat), _f64(w)
    pins, assign, part_sizes, node_size = _i32(pins), _i32(assign), _i64(part_sizes), _i32(node_size)
    n = len(inc_off) - 1
    K = pins.shape[1] if pins.ndim == 2 else 0
    target = np.zeros(max(n, 1), dtype=np.int32)
    gain = np.zeros(max(n, 1), dtype=np.float64)
    rc = _lib.load().dhgp_propose_moves(
        C.c_int32(n), _lib.ptr(inc_off), _lib.ptr(inc_dat), C.c_int32(len(pin_off) - 1), _lib.ptr(pin_off),
        _lib.ptr(pin_dat), _lib.ptr(w), _lib.ptr(pins), C.c_int32(K), _lib.ptr(assign), _lib.ptr(part_sizes),
        _lib.ptr(node_size), C.c_int64(int(max_size)), _dev(), _lib.ptr(target), _lib.ptr(gain))
    _lib.raise_for(rc)
    return target[:n], gain[:n]


def sequence_gains(inc_off, inc_dat, pin_off, pin_dat, w, pins, node, from_part, to_part, gain_iso, pos):
    inc_off, inc_dat, pin_off, pin_dat, w = _i64(inc_off), _i32(inc_dat), _i64(pin_off), _i32(pin_dat), _f64(w)
    pins, node, from_part, to_part = _i32(pins), _i32(node), _i32(from_part), _i32(to_part)
    gain_iso, pos = _f64(gain_iso), _i64(pos)
    m = len(node)
    out = np.zeros(max(m, 1), dtype=np.float64)
    rc = _lib.load().dhgp_sequence_gains(
        C.c_int32(len(inc_off) - 1), _lib.ptr(inc_off), _lib.ptr(inc_dat), C.c_int32(len(pin_off) - 1),
        _lib.ptr(pin_off), _lib.ptr(pin_dat), _lib.ptr(w), _lib.ptr(pins), C.c_int32(pins.shape[1]),
        C.c_int32(m), _lib.ptr(node), _lib.ptr(from_part), _lib.ptr(to_part), _lib.ptr(gain_iso), _lib.ptr(pos),
        _dev(), _lib.ptr(out))
    _lib.raise_for(rc)
    return out[:m]


def build_events_and_select(num_nodes, in_off, in_dat, node_size, node, from_part, to_part, gain_seq, pins_in,
                            part_sizes, part_inbound, max_size, max_inbound):
    """refine.build_events_and_select (refine.py:178-247) over explicit
    arrays: the dense pins_in matrix (E x K) as in the reference.  Returns
    (k, total_gain, active)."""
    in_off, in_dat, node_size = _i64(in_off), _i32(in_dat), _i32(node_size)
    node, from_part, to_part, gain_seq = _i32(node), _i32(from_part), _i32(to_part), _f64(gain_seq)
    pins_in, part_sizes, part_inbound = _i32(pins_in), _i64(part_sizes), _i64(part_inbound)
    m = len(node)
    active = np.zeros(m + 1, dtype=np.int64)
    k = C.c_int64(0)
    tg = C.c_double(0.0)
    rc = _lib.load().dhgp_build_events_and_select(
        C.c_int32(num_nodes), _lib.ptr(in_off), _lib.ptr(in_dat), _lib.ptr(node_size), C.c_int32(pins_in.shape[0]),
        C.c_int32(pins_in.shape[1]), C.c_int32(m), _lib.ptr(node), _lib.ptr(from_part), _lib.ptr(to_part),
        _lib.ptr(gain_seq), _lib.ptr(pins_in), _lib.ptr(part_sizes), _lib.ptr(part_inbound), C.c_int64(max_size),
        C.c_int64(max_inbound), _dev(), C.byref(k), C.byref(tg), _lib.ptr(active))
    _lib.raise_for(rc)
    return int(k.value), float(tg.value), active


__all__ = [
    "available_backends", "active_backend", "set_backend", "get_module", "union_size_sorted",
    "fill_histograms", "select_first_valid", "resolve_matching", "connectivity_value", "compute_pins",
    "propose_moves", "sequence_gains", "build_events_and_select", "DhgError",
]
