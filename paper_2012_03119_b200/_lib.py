"""ctypes bindings of libtsg.so (include/tsg.h).

The product has exactly one compute path: the CUDA library.  If the library
is missing or no CUDA device is present, every compute call raises -- there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSG_LIB", os.path.join(HERE, "libtsg.so"))

TSG_OK, TSG_EINVAL, TSG_ECAPACITY, TSG_ERANGE, TSG_ECUDA, TSG_ENOMEM = range(6)
TSG_F_TIMING = 1
TSG_F_ALL_PAIRS = 2
TSG_F_CHUNK_FILTER = 4


class CapacityError(ValueError):
    """More assignments or groups than the configured word width holds
    (bitpack.py:28-29)."""


class TsgError(RuntimeError):
    """CUDA-side failure (no device, launch error, out of memory)."""


class tsg_config(C.Structure):
    _fields_ = [("lane_width", C.c_int32), ("group_width", C.c_int32), ("device", C.c_int32),
                ("flags", C.c_int32), ("report_capacity", C.c_int64)]


class tsg_round_result(C.Structure):
    _fields_ = [("reports", C.c_int64), ("clauses_tested", C.c_int64), ("aggregate_tests", C.c_int64),
                ("aggregate_tests_negative", C.c_int64), ("lane_tests", C.c_int64),
                ("lane_triggers", C.c_int64), ("n_chunks", C.c_int32), ("reruns", C.c_int32),
                ("encode_ms", C.c_double), ("test_ms", C.c_double), ("chunk_positives", C.c_int64)]


class tsg_counters_t(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "rounds", "reports", "clauses_tested", "aggregate_tests", "aggregate_tests_negative", "lane_tests",
        "lane_triggers", "reruns", "clauses_added", "clauses_removed", "clauses_deleted", "reduces")]


from .reports import RECORD_DTYPE as REPORT_DTYPE  # noqa: E402  (tsg_report, 16 bytes)

# every symbol include/tsg.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "tsg_last_error", "tsg_abi_version", "tsg_device_count", "tsg_create", "tsg_destroy",
    "tsg_add_clauses", "tsg_store_size", "tsg_bucket_count", "tsg_bucket_info", "tsg_bucket_read",
    "tsg_scale_activities", "tsg_reduce", "tsg_remove_clauses", "tsg_stage_snapshots", "tsg_round",
    "tsg_round_prepare", "tsg_round_encode", "tsg_round_tables", "tsg_round_test", "tsg_fetch_reports",
    "tsg_reports_device", "tsg_sync", "tsg_stream", "tsg_pack", "tsg_aggregate", "tsg_lane_trigger",
    "tsg_aggregate_trigger", "tsg_packed_words", "tsg_pack_rows", "tsg_stage_packed",
    "tsg_fetch_reports_async", "tsg_fetch_wait", "tsg_round_launch", "tsg_round_collect",
    "tsg_set_record_bytes", "tsg_get_clauses", "tsg_counters", "tsg_set_timing", "tsg_round_encode_groups",
    "tsg_round_layout", "tsg_set_all_pairs", "tsg_round_tables_copy", "tsg_reduce_begin", "tsg_reduce_hist",
    "tsg_reduce_commit", "tsg_fetch_ordered", "tsg_stage_packed_segments", "tsg_host_alloc", "tsg_host_free",
    "tsg_device_alloc", "tsg_device_free", "tsg_ingress_copy", "tsg_ring_open", "tsg_ring_close",
    "tsg_ring_drain", "tsg_ring_status", "tsg_stage_packed_mixed",
)

_lib = None
_lock = threading.Lock()


def _declare(L):
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    pI64 = C.POINTER(C.c_int64)
    sig = {
        "tsg_last_error": ([], C.c_char_p),
        "tsg_abi_version": ([], C.c_int),
        "tsg_device_count": ([C.POINTER(C.c_int32)], C.c_int),
        "tsg_create": ([I32, C.POINTER(tsg_config), C.POINTER(P)], C.c_int),
        "tsg_destroy": ([P], C.c_int),
        "tsg_add_clauses": ([P, P, P, I64, P, P, D], C.c_int),
        "tsg_store_size": ([P, pI64], C.c_int),
        "tsg_bucket_count": ([P, C.POINTER(C.c_int32)], C.c_int),
        "tsg_bucket_info": ([P, I32, C.POINTER(C.c_int32), pI64], C.c_int),
        "tsg_bucket_read": ([P, I32, P, P, P, P], C.c_int),
        "tsg_scale_activities": ([P, D], C.c_int),
        "tsg_get_clauses": ([P, P, I64, P, P, I64, pI64], C.c_int),
        "tsg_counters": ([P, P], C.c_int),
        "tsg_set_timing": ([P, I32], C.c_int),
        "tsg_set_all_pairs": ([P, I32], C.c_int),
        "tsg_round_tables_copy": ([P, P], C.c_int),
        "tsg_round_encode_groups": ([P, I32, I32, I32], C.c_int),
        "tsg_round_layout": ([P, pI64, pI64, pI64, pI64], C.c_int),
        "tsg_reduce": ([P, I64, I64, pI64, P], C.c_int),
        "tsg_reduce_begin": ([P, I64, pI64], C.c_int),
        "tsg_fetch_ordered": ([P, I32, P, I32, P, I32, P, I32, P, P, I64, pI64], C.c_int),
        "tsg_stage_packed_segments": ([P, P, P, I32, I64], C.c_int),
        "tsg_host_alloc": ([I64, C.POINTER(P)], C.c_int),
        "tsg_host_free": ([P], C.c_int),
        "tsg_device_alloc": ([P, I64, C.POINTER(P)], C.c_int),
        "tsg_device_free": ([P, P], C.c_int),
        "tsg_ingress_copy": ([P, P, P, I64], C.c_int),
        "tsg_ring_open": ([P, I64, I64], C.c_int),
        "tsg_ring_close": ([P], C.c_int),
        "tsg_ring_drain": ([P, P, I64, pI64, I64, pI64], C.c_int),
        "tsg_ring_status": ([P, pI64, pI64, C.POINTER(I32)], C.c_int),
        "tsg_stage_packed_mixed": ([P, P, I64, I64, P, I64, I64], C.c_int),
        "tsg_reduce_hist": ([P, C.c_uint64, C.c_uint64, I32, P], C.c_int),
        "tsg_reduce_commit": ([P, C.c_uint64, C.c_uint64, I32, pI64, P, I64], C.c_int),
        "tsg_remove_clauses": ([P, P, I64, pI64], C.c_int),
        "tsg_stage_snapshots": ([P, P, I64, I64, I32], C.c_int),
        "tsg_packed_words": ([I32, P], C.c_int),
        "tsg_pack_rows": ([P, I64, I64, I32, P, I64], C.c_int),
        "tsg_stage_packed": ([P, P, I64, I64, I32], C.c_int),
        "tsg_round": ([P, P, P, I32, D, C.POINTER(tsg_round_result)], C.c_int),
        "tsg_round_prepare": ([P, P, P, I32], C.c_int),
        "tsg_round_encode": ([P], C.c_int),
        "tsg_round_tables": ([P, C.POINTER(P), pI64], C.c_int),
        "tsg_round_test": ([P, D, C.POINTER(tsg_round_result)], C.c_int),
        "tsg_fetch_reports": ([P, P, I64, pI64], C.c_int),
        "tsg_fetch_reports_async": ([P, P, I64, pI64], C.c_int),
        "tsg_fetch_wait": ([P], C.c_int),
        "tsg_set_record_bytes": ([P, I32], C.c_int),
        "tsg_round_launch": ([P, D], C.c_int),
        "tsg_round_collect": ([P, C.POINTER(tsg_round_result)], C.c_int),
        "tsg_reports_device": ([P, C.POINTER(P), pI64], C.c_int),
        "tsg_sync": ([P], C.c_int),
        "tsg_stream": ([P, C.POINTER(P)], C.c_int),
        "tsg_pack": ([I32, P, I64, I64, I32, I32, P, P], C.c_int),
        "tsg_aggregate": ([I32, P, P, P, I32, I32, I32, P, P, P], C.c_int),
        "tsg_lane_trigger": ([I32, P, P, I32, I32, C.c_uint64, P, P, I64, P], C.c_int),
        "tsg_aggregate_trigger": ([I32, P, P, P, I32, I32, I32, P, P, I64, P], C.c_int),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("TSG_LIB") and not hasattr(L, name):
            continue  # an older library loaded for a side-by-side measurement
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def load(path: str = LIB_PATH):
    """Load libtsg.so (building it first if the sources are newer)."""
    global _lib
    with _lock:
        if _lib is None:
            from . import build as _build
            if not os.path.exists(path):
                _build.build()
            L = C.CDLL(path)
            _declare(L)
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == TSG_OK:
        return
    msg = (load().tsg_last_error() or b"").decode(errors="replace")
    if rc == TSG_EINVAL:
        raise ValueError(msg)
    if rc == TSG_ECAPACITY:
        raise CapacityError(msg)
    if rc == TSG_ERANGE:
        raise IndexError(msg)
    if rc == TSG_ENOMEM:
        raise MemoryError(msg)
    raise TsgError(msg)


def ptr(a):
    """Raw pointer of a numpy array (or None)."""
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


def device_count() -> int:
    n = C.c_int32(0)
    load().tsg_device_count(C.byref(n))
    return n.value
