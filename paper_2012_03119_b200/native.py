"""Thin object wrapper of one C-ABI engine handle (include/tsg.h).

Used by the Engine mirror's bulk paths, bench.py and the multi-GPU runner:
bulk clause ingest from flat arrays, snapshot staging from host or device
memory, split encode/test for table broadcast, record fetch.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Tuple

import numpy as np

from . import _lib, reports
from ._lib import REPORT_DTYPE, check, ptr


def packed_words(num_vars: int) -> int:
    """u64 words per packed snapshot row (include/tsg.h tsg_packed_words)."""
    w = C.c_int64(0)
    check(_lib.load().tsg_packed_words(num_vars, C.byref(w)))
    return w.value


def pack_rows(rows: np.ndarray, num_vars: int, out: Optional[np.ndarray] = None, threads: int = 1) -> np.ndarray:
    """int8 snapshot rows [n, >= num_vars+1] -> packed rows uint64[n, packed_words]
    (2 bits per variable; tsg_pack_rows, GIL released).  A round's worth of
    rows is split over the library's host worker pool inside the one call
    (the packing is bound by host memory bandwidth); `threads` is accepted
    for compatibility and no longer used."""
    rows = np.ascontiguousarray(rows, np.int8)
    n = rows.shape[0]
    w = packed_words(num_vars)
    if out is None:
        out = np.empty((n, w), np.uint64)
    if n:
        check(_lib.load().tsg_pack_rows(C.c_void_p(rows.ctypes.data), n, rows.strides[0], num_vars,
                                        C.c_void_p(out.ctypes.data), out.strides[0] // 8))
    return out


class NativeEngine:
    def __init__(self, num_vars: int, lane_width: int = 32, group_width: int = 32, device: int = 0,
                 timing: bool = False, report_capacity: int = 0, chunk_filter: bool = False):
        self.L = _lib.load()
        self.num_vars = num_vars
        self.lane_width, self.group_width = lane_width, group_width
        cfg = _lib.tsg_config(lane_width, group_width, device,
                              (_lib.TSG_F_TIMING if timing else 0) | (_lib.TSG_F_CHUNK_FILTER if chunk_filter else 0),
                              report_capacity)
        h = C.c_void_p()
        check(self.L.tsg_create(num_vars, C.byref(cfg), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.tsg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- store -----------------------------------------------------------
    def add_clauses(self, flat: np.ndarray, offsets: np.ndarray, ids: np.ndarray,
                    origins: Optional[np.ndarray] = None, activity: float = 1.0) -> None:
        n = len(offsets) - 1
        if origins is None:
            origins = np.zeros(n, np.int32)
        flat = np.ascontiguousarray(flat, np.int32)
        if flat.size == 0:
            flat = np.zeros(1, np.int32)
        check(self.L.tsg_add_clauses(self.h, ptr(flat), ptr(np.ascontiguousarray(offsets, np.int64)), n,
                                     ptr(np.ascontiguousarray(ids, np.int64)),
                                     ptr(np.ascontiguousarray(origins, np.int32)), activity))

    def __len__(self) -> int:
        n = C.c_int64(0)
        check(self.L.tsg_store_size(self.h, C.byref(n)))
        return n.value

    def buckets(self):
        """[(size, lits[count,size], ids, origins, acts)] in creation order."""
        nb = C.c_int32(0)
        check(self.L.tsg_bucket_count(self.h, C.byref(nb)))
        out = []
        for b in range(nb.value):
            s, n = C.c_int32(0), C.c_int64(0)
            check(self.L.tsg_bucket_info(self.h, b, C.byref(s), C.byref(n)))
            lits = np.zeros((n.value, s.value), np.int32)
            ids = np.zeros(n.value, np.int64)
            org = np.zeros(n.value, np.int32)
            acts = np.zeros(n.value, np.float64)
            if n.value:
                check(self.L.tsg_bucket_read(self.h, b, ptr(lits), ptr(ids), ptr(org), ptr(acts)))
            out.append((s.value, lits, ids, org, acts))
        return out

    def reduce(self, eligible_below: int, target: int) -> np.ndarray:
        removed = C.c_int64(0)
        ids = np.zeros(max(target, 1), np.int64)
        check(self.L.tsg_reduce(self.h, eligible_below, target, C.byref(removed), ptr(ids)))
        return ids[:removed.value]

    # split reduce selection over shards (sharded.global_reduce)
    def reduce_begin(self, eligible_below: int) -> int:
        n = C.c_int64(0)
        check(self.L.tsg_reduce_begin(self.h, eligible_below, C.byref(n)))
        return n.value

    def reduce_hist(self, prefix_hi: int, prefix_lo: int, bits: int) -> np.ndarray:
        h = np.zeros(256, np.uint64)
        check(self.L.tsg_reduce_hist(self.h, C.c_uint64(prefix_hi), C.c_uint64(prefix_lo), bits, ptr(h)))
        return h

    def reduce_commit(self, prefix_hi: int, prefix_lo: int, bits: int) -> np.ndarray:
        n = max(len(self), 1)
        ids = np.zeros(n, np.int64)
        removed = C.c_int64(0)
        check(self.L.tsg_reduce_commit(self.h, C.c_uint64(prefix_hi), C.c_uint64(prefix_lo), bits, C.byref(removed),
                                       ptr(ids), n))
        return ids[:removed.value]

    def remove(self, ids) -> int:
        a = np.ascontiguousarray(ids, np.int64)
        removed = C.c_int64(0)
        check(self.L.tsg_remove_clauses(self.h, ptr(a if a.size else np.zeros(1, np.int64)), a.size,
                                        C.byref(removed)))
        return removed.value

    def get_clauses(self, ids) -> list:
        """Literal tuples of the stored clauses `ids` (None where not stored), in
        their original order (tsg_get_clauses; engine.py:165-169)."""
        q = np.ascontiguousarray(ids, np.int64)
        n = len(q)
        if n == 0:
            return []
        sizes = np.zeros(n, np.int32)
        tot = C.c_int64(0)
        check(self.L.tsg_get_clauses(self.h, ptr(q), n, ptr(sizes), None, 0, C.byref(tot)))
        lits = np.zeros(max(tot.value, 1), np.int32)
        check(self.L.tsg_get_clauses(self.h, ptr(q), n, ptr(sizes), ptr(lits), len(lits), C.byref(tot)))
        out, o = [], 0
        for s in sizes.tolist():
            if s < 0:
                out.append(None)
            else:
                out.append(tuple(lits[o:o + s].tolist()))
                o += s
        return out

    def set_all_pairs(self, on: bool) -> None:
        """Emit every triggering (clause, group) -- multi_trigger's pair set --
        instead of the first per (clause, thread) (tsg_set_all_pairs)."""
        check(self.L.tsg_set_all_pairs(self.h, 1 if on else 0))

    def tables_from(self, src: "NativeEngine") -> None:
        """Copy src's encoded round tables into this engine over NVLink
        (tsg_round_tables_copy); both have prepared the same round."""
        check(self.L.tsg_round_tables_copy(self.h, src.h))

    def set_timing(self, every: int) -> None:
        """With timing=True: events on every `every`-th round only (tsg_set_timing)."""
        check(self.L.tsg_set_timing(self.h, every))

    def counters(self) -> dict:
        """Cumulative figures (tsg_counters)."""
        c = _lib.tsg_counters_t()
        check(self.L.tsg_counters(self.h, C.byref(c)))
        return {n: getattr(c, n) for n, _ in c._fields_}

    def scale(self, factor: float) -> None:
        check(self.L.tsg_scale_activities(self.h, factor))

    # ---- round ------------------------------------------------------------
    def stage(self, rows: np.ndarray) -> None:
        rows = np.ascontiguousarray(rows, np.int8)
        check(self.L.tsg_stage_snapshots(self.h, ptr(rows), rows.shape[0], rows.shape[1], 0))

    def stage_device(self, dptr: int, n_rows: int, pitch: int) -> None:
        check(self.L.tsg_stage_snapshots(self.h, C.c_void_p(dptr), n_rows, pitch, 1))

    def stage_packed(self, packed: np.ndarray) -> None:
        """Packed rows (pack_rows) from host memory (pinned memory copies fastest)."""
        check(self.L.tsg_stage_packed(self.h, C.c_void_p(packed.ctypes.data), packed.shape[0],
                                      packed.strides[0] // 8, 0))

    def stage_packed_mixed(self, packed: np.ndarray, raw: np.ndarray) -> None:
        """Rows 0..len(packed)-1 packed on the host (pack_rows), the rest as
        int8 rows, packed on the device (tsg_stage_packed_mixed).  Both
        arrays must stay unchanged until the round is collected."""
        packed = np.ascontiguousarray(packed, np.uint64)
        raw = np.ascontiguousarray(raw, np.int8)
        np_, nr = (packed.shape[0] if packed.size else 0), (raw.shape[0] if raw.size else 0)
        check(self.L.tsg_stage_packed_mixed(self.h, ptr(packed) if np_ else None, np_,
                                            packed.shape[1] if np_ else packed_words(self.num_vars),
                                            ptr(raw) if nr else None, nr, raw.strides[0] if nr else self.num_vars + 1))

    def stage_packed_ptr(self, ptr_: int, n_rows: int, pitch_words: int, on_device: bool) -> None:
        check(self.L.tsg_stage_packed(self.h, C.c_void_p(ptr_), n_rows, pitch_words, 1 if on_device else 0))

    def prepare(self, group_lanes, group_tid) -> None:
        self._gl = np.ascontiguousarray(group_lanes, np.int32)
        self._gt = np.ascontiguousarray(group_tid, np.int32)
        check(self.L.tsg_round_prepare(self.h, ptr(self._gl), ptr(self._gt), len(self._gl)))

    def encode(self) -> None:
        check(self.L.tsg_round_encode(self.h))

    def encode_groups(self, g_begin: int, g_end: int, sentinel: bool) -> None:
        """Encode groups [g_begin, g_end) from rows holding only those groups
        (tsg_round_encode_groups; split ingress across GPUs)."""
        check(self.L.tsg_round_encode_groups(self.h, g_begin, g_end, 1 if sentinel else 0))

    def layout(self) -> Tuple[int, int, int, int]:
        """(agg_off, agg_len, lane_off, group_bytes) inside tables() (tsg_round_layout)."""
        v = [C.c_int64(0) for _ in range(4)]
        check(self.L.tsg_round_layout(self.h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def tables(self) -> Tuple[int, int]:
        p, n = C.c_void_p(), C.c_int64(0)
        check(self.L.tsg_round_tables(self.h, C.byref(p), C.byref(n)))
        return p.value or 0, n.value

    def test(self, activity_inc: float = 1.0) -> _lib.tsg_round_result:
        res = _lib.tsg_round_result()
        check(self.L.tsg_round_test(self.h, activity_inc, C.byref(res)))
        return res

    def launch(self, activity_inc: float = 1.0) -> None:
        """Queue the test of the prepared, encoded round (tsg_round_launch)."""
        check(self.L.tsg_round_launch(self.h, activity_inc))

    def collect(self) -> _lib.tsg_round_result:
        """Figures of the launched round (tsg_round_collect)."""
        res = _lib.tsg_round_result()
        check(self.L.tsg_round_collect(self.h, C.byref(res)))
        return res

    def round(self, group_lanes, group_tid, activity_inc: float = 1.0) -> _lib.tsg_round_result:
        gl = np.ascontiguousarray(group_lanes, np.int32)
        gt = np.ascontiguousarray(group_tid, np.int32)
        res = _lib.tsg_round_result()
        check(self.L.tsg_round(self.h, ptr(gl), ptr(gt), len(gl), activity_inc, C.byref(res)))
        return res

    record_bytes = 16

    def set_record_bytes(self, nbytes: int) -> None:
        """Egress record format: 16 (tsg_report), 12 (lane_width <= 32) or 8
        (also engine ids < 2^27 and <= 32 groups)."""
        check(self.L.tsg_set_record_bytes(self.h, nbytes))
        self.record_bytes = nbytes

    def fetch_raw(self, n: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """The round's records in the egress format (tsg_report, or 12-byte)."""
        if out is None or len(out) < n:
            out = np.zeros(max(n, 1), {16: REPORT_DTYPE, 12: reports.RECORD12_DTYPE,
                                       8: reports.RECORD8_DTYPE}[self.record_bytes])
        got = C.c_int64(0)
        if n:
            check(self.L.tsg_fetch_reports(self.h, ptr(out), n, C.byref(got)))
        return out[:got.value]

    def fetch_async(self, out: np.ndarray) -> int:
        """Start copying the round's records into `out` (pinned, REPORT_DTYPE);
        returns the count.  Valid after wait()."""
        got = C.c_int64(0)
        check(self.L.tsg_fetch_reports_async(self.h, ptr(out), len(out), C.byref(got)))
        return got.value

    def wait(self) -> None:
        check(self.L.tsg_fetch_wait(self.h))

    def fetch(self, n: int) -> np.ndarray:
        """Decoded records: (engine_id, group, lane_mask), unordered."""
        return reports.decode(self.fetch_raw(n))

    # ---- host report ring (tsg_ring_*) ----------------------
    def ring_open(self, capacity: int = 1 << 20, wait_ms: float = 2000.0) -> None:
        """Records of the rounds launched from now on go straight into a
        page-locked host ring, drained with ring_drain while the kernel runs."""
        check(self.L.tsg_ring_open(self.h, int(capacity), max(1, int(wait_ms * 1000))))

    def ring_close(self) -> None:
        check(self.L.tsg_ring_close(self.h))

    def ring_drain(self, max_records: int = 1 << 16, timeout_ms: float = 0.0,
                   out: Optional[np.ndarray] = None, with_pos: bool = False):
        """One contiguous run of landed records, in ring order (raw
        REPORT_DTYPE); empty after timeout_ms with none.  with_pos: also the
        ring position of the first (records are numbered from the ring's
        opening, rounds in launch order).  Safe to call from threads other
        than the one running the rounds (ctypes releases the GIL)."""
        if out is None or len(out) < max_records:
            out = np.zeros(max(1, max_records), REPORT_DTYPE)
        got, pos = C.c_int64(0), C.c_int64(-1)
        check(self.L.tsg_ring_drain(self.h, ptr(out), max_records, C.byref(got), int(timeout_ms * 1000),
                                    C.byref(pos)))
        return (out[:got.value], pos.value) if with_pos else out[:got.value]

    def ring_status(self):
        """(records of the collected rounds, records drained, dropped?)"""
        e, c, f = C.c_int64(0), C.c_int64(0), C.c_int32(0)
        check(self.L.tsg_ring_status(self.h, C.byref(e), C.byref(c), C.byref(f)))
        return e.value, c.value, bool(f.value)

    def sync(self) -> None:
        check(self.L.tsg_sync(self.h))

    def stream(self) -> int:
        s = C.c_void_p()
        check(self.L.tsg_stream(self.h, C.byref(s)))
        return s.value or 0


class RingDrainer:
    """CPU threads draining an engine's host report ring (tsg_ring_drain)
    while its rounds run -- the consumer side of north_star subsystem 4.
    Each drained run carries its ring position, so `take(n)` returns exactly
    the next n records in ring order -- the next round's when n is that
    round's report count -- however many threads drain and however many
    rounds are in flight."""

    def __init__(self, eng: NativeEngine, threads: int = 1, batch: int = 1 << 16):
        import threading
        self.eng = eng
        self._runs: dict = {}   # ring position -> records landed from there
        self._next = 0          # position of the next record take() hands out
        self._lock = threading.Lock()
        self._cv = threading.Condition(self._lock)
        self._stop = threading.Event()
        self.error: Optional[BaseException] = None
        self._threads = [threading.Thread(target=self._run, args=(batch,), daemon=True) for _ in range(threads)]
        for t in self._threads:
            t.start()

    def _run(self, batch: int) -> None:
        buf = np.empty(batch, REPORT_DTYPE)
        try:
            while not self._stop.is_set():
                got, pos = self.eng.ring_drain(batch, timeout_ms=1.0, out=buf, with_pos=True)
                if len(got):
                    with self._cv:
                        self._runs[pos] = got  # a view of buf: a fresh buf follows
                        self._cv.notify_all()
                    buf = np.empty(batch, REPORT_DTYPE)
        except BaseException as e:  # surfaced by take()
            with self._cv:
                self.error = e
                self._cv.notify_all()

    def _ready(self) -> int:
        """Records available contiguously from self._next (lock held)."""
        k, pos = 0, self._next
        while pos in self._runs:
            k += len(self._runs[pos])
            pos += len(self._runs[pos])
        return k

    def take(self, n: int, timeout_s: float = 60.0) -> np.ndarray:
        """The next n records in ring order (blocks until drained)."""
        import time
        end = time.monotonic() + timeout_s
        with self._cv:
            while self._ready() < n and self.error is None:
                left = end - time.monotonic()
                if left <= 0:
                    raise TimeoutError(f"ring drained {self._ready()} of {n} records")
                self._cv.wait(min(left, 0.1))
            if self.error is not None:
                raise self.error
            parts, got = [], 0
            while got < n:
                run = self._runs.pop(self._next)
                use = min(len(run), n - got)
                parts.append(run[:use])
                if use < len(run):  # the rest starts the next take
                    self._runs[self._next + use] = run[use:]
                self._next += use
                got += use
            return parts[0] if len(parts) == 1 else (np.concatenate(parts) if parts else np.zeros(0, REPORT_DTYPE))

    def close(self) -> None:
        self._stop.set()
        for t in self._threads:
            t.join()

