"""ctypes binding of libdhgp.so (include/dhgp.h).

The library is loaded lazily so that the package imports on a machine
without a GPU (for the CPU test tier); every compute entry point raises
:class:`CudaUnavailableError` when the library is missing or no CUDA device
is visible.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libdhgp.so"
if os.environ.get("DHGP_LIB_VARIANT"):  # diagnostics: an in-tree A/B build, libdhgp_<variant>.so
    LIB_PATH = LIB_PATH.with_name(f"libdhgp_{os.environ['DHGP_LIB_VARIANT']}.so")

# status codes (include/dhgp.h)
OK = 0
ERR_INFEASIBLE = 1
ERR_MAX_LEVELS = 2
ERR_MATCHING = 3
ERR_INVALID_RESULT = 4
ERR_CUDA = 5
ERR_ARG = 6
ERR_UNSUPPORTED = 7


class CudaUnavailableError(RuntimeError):
    """libdhgp.so is not built or no CUDA device is visible."""


class DhgpGraph(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int32), ("num_edges", C.c_int32),
        ("edge_weight", C.c_void_p),
        ("src_off", C.c_void_p), ("src_dat", C.c_void_p),
        ("dst_off", C.c_void_p), ("dst_dat", C.c_void_p),
        ("node_size", C.c_void_p),
    ]


class DhgpConfig(C.Structure):
    _fields_ = [
        ("max_size", C.c_int64), ("max_inbound", C.c_int64),
        ("max_rounds", C.c_int32), ("batch_size", C.c_int32), ("max_levels", C.c_int32),
        ("device", C.c_int32),
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


OBSERVER = C.CFUNCTYPE(None, C.POINTER(DhgpEvent), C.c_void_p)

# every symbol include/dhgp.h declares for libdhgp.so
EXPORTS = [
    "dhgp_last_error", "dhgp_build_info", "dhgp_device_count", "dhgp_partition", "dhgp_stats_free",
    "dhgp_session_create", "dhgp_session_partition", "dhgp_session_destroy", "dhgp_session_kernel_stats",
    "dhgp_session_set_profiling", "dhgp_incidence", "dhgp_neighbors", "dhgp_free", "dhgp_check_feasibility",
    "dhgp_evaluate", "dhgp_baseline", "dhgp_union_size_sorted", "dhgp_fill_histograms", "dhgp_select_first_valid",
    "dhgp_resolve_matching", "dhgp_connectivity_value", "dhgp_compute_pins", "dhgp_propose_moves",
    "dhgp_sequence_gains", "dhgp_build_events_and_select",
    "dhgp_comm_nccl_unique_id", "dhgp_comm_init_nccl", "dhgp_comm_init_host", "dhgp_comm_set_min_units",
    "dhgp_comm_stats", "dhgp_comm_destroy", "dhgp_partition_sharded", "dhgp_session_set_comm", "dhgp_shard_range",
    "dhgp_parse_dhg_begin", "dhgp_parse_dhg_slow_lines", "dhgp_parse_dhg_finish", "dhgp_parse_dhg_fetch",
    "dhgp_parse_dhg_line_range", "dhgp_parse_free",
]

_lib = None
_device_checked = False


def load(require_device: bool = True):
    """Return the loaded library; raise loudly when it cannot run."""
    global _lib, _device_checked
    if _lib is None:
        if not LIB_PATH.exists():
            raise CudaUnavailableError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` (or `make`)"
            )
        L = C.CDLL(str(LIB_PATH))
        L.dhgp_last_error.restype = C.c_char_p
        L.dhgp_build_info.restype = C.c_char_p
        L.dhgp_comm_destroy.argtypes = [C.c_void_p]
        L.dhgp_comm_destroy.restype = None
        L.dhgp_parse_free.argtypes = [C.c_void_p]
        L.dhgp_parse_free.restype = None
        _lib = L
    if require_device and not _device_checked:
        n = C.c_int32(0)
        rc = _lib.dhgp_device_count(C.byref(n))
        if rc != OK or n.value < 1:
            raise CudaUnavailableError("no CUDA device visible to libdhgp.so (there is no CPU fallback)")
        _device_checked = True
    return _lib


def device() -> int:
    return int(os.environ.get("DHGP_DEVICE", "0"))


def ptr(a: np.ndarray | None):
    return None if a is None else C.c_void_p(a.ctypes.data)


def c_arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def take(p, n: int, dtype) -> np.ndarray:
    if n <= 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dtype, copy=True)


def raise_for(rc: int) -> None:
    """Map a status code onto the reference exception hierarchy (errors.py)."""
    if rc == OK:
        return
    from .errors import DhgError, InfeasibleError, MatchingInvariantError

    msg = _lib.dhgp_last_error().decode() if _lib is not None else ""
    if rc == ERR_INFEASIBLE:
        raise InfeasibleError(msg)
    if rc == ERR_MATCHING:
        raise MatchingInvariantError(msg)
    if rc in (ERR_MAX_LEVELS, ERR_INVALID_RESULT):
        raise DhgError(msg)
    if rc == ERR_ARG:
        raise ValueError(msg)
    if rc == ERR_UNSUPPORTED:
        raise DhgError(f"unsupported input: {msg}")
    raise RuntimeError(f"libdhgp CUDA error: {msg}")
