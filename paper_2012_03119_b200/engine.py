"""The clause-exchange engine on a B200: drop-in for triggersat.engine.Engine.

Same public surface as the reference (engine.py:44-525): ``EngineConfig``,
``AssignmentSnapshot``, ``Report``, ``RoundResult``, ``RoundTrace`` and
``Engine`` with ``add_clause`` / ``submit_assignment`` / ``drain_reports`` /
``run_round`` / ``reduce_store`` / ``serve`` / ``raw_counters`` / ``store`` /
``counters`` / ``trace`` / ``config``.  The host keeps what the reference
keeps on its producer side -- the id lock, the staging list, the per-thread
snapshot and report queues (engine.py:273-279) -- and the clause store lives
in HBM behind the C ABI (include/tsg.h): size buckets, activities, ids and
the round's kernels.  The only host copy of clause data is the literal tuple
per engine id that Reports carry (engine.py:90-102).

There is no CPU path: constructing an Engine without the CUDA library or a
CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import itertools
import threading
import time
from collections import deque
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from . import reports as _reports
from ._lib import REPORT_DTYPE, check, ptr

#: Activities are rescaled when the bump increment passes this (engine.py:39-40).
_ACTIVITY_RESCALE = 1e100


@dataclass
class EngineConfig:
    """Tunables, identical to the reference (engine.py:44-74) plus the device
    ordinal and the initial report-buffer size."""

    max_clauses: int = 5_000_000
    assignment_queue_capacity: Optional[int] = None
    lane_width: int = 32
    group_width: int = 32
    activity_decay: float = 0.999
    reduce_keep_fraction: float = 0.5
    interleave_stride: int = 32
    trace: bool = False
    device: int = 0
    report_capacity: int = 0
    timing: bool = False

    def __post_init__(self):
        if self.max_clauses < 1:
            raise ValueError("max_clauses must be >= 1")
        if not 0 < self.activity_decay <= 1:
            raise ValueError("activity_decay must be in (0, 1]")
        if not 0 < self.reduce_keep_fraction < 1:
            raise ValueError("reduce_keep_fraction must be in (0, 1)")
        if self.assignment_queue_capacity is None:
            self.assignment_queue_capacity = 2 * self.lane_width
        if self.assignment_queue_capacity < 1:
            raise ValueError("assignment_queue_capacity must be >= 1")


@dataclass
class AssignmentSnapshot:
    """One thread's trail at a propagation fixpoint (engine.py:77-87)."""

    thread_id: int
    values: np.ndarray
    seq: int


@dataclass
class Report:
    """A stored clause that triggered for ``destination`` (engine.py:90-102)."""

    destination: int
    lits: tuple
    engine_id: int
    lane_mask: int


@dataclass
class _ReportBatch:
    """One round's reports for one destination, in emission order."""

    lits: list
    eids: list
    masks: list


@dataclass
class RoundResult:
    reports_emitted: int = 0
    clauses_tested: int = 0
    assignments_consumed: int = 0
    aggregate_tests_negative: int = 0


@dataclass
class RoundTrace:
    snapshots: list
    store: list
    reports: list


class BucketView:
    """Live view of one device size bucket (the reference's _SizeBucket,
    engine.py:122-200).  Every attribute read fetches from HBM."""

    def __init__(self, engine: "Engine", index: int, size: int):
        self._e, self.index, self.size = engine, index, size

    @property
    def count(self) -> int:
        s = C.c_int32(0)
        n = C.c_int64(0)
        check(self._e._L.tsg_bucket_info(self._e._h, self.index, C.byref(s), C.byref(n)))
        return n.value

    def _read(self, lits=False, ids=False, origins=False, acts=False):
        n = self.count
        out = [np.zeros((n, self.size), np.int32) if lits else None,
               np.zeros(n, np.int64) if ids else None,
               np.zeros(n, np.int32) if origins else None,
               np.zeros(n, np.float64) if acts else None]
        if n:
            check(self._e._L.tsg_bucket_read(self._e._h, self.index, *(ptr(a) for a in out)))
        return out

    @property
    def activities(self) -> np.ndarray:
        return self._read(acts=True)[3]

    @property
    def engine_ids(self) -> np.ndarray:
        return self._read(ids=True)[1]

    @property
    def origins(self) -> np.ndarray:
        return self._read(origins=True)[2]

    def lits_at(self, slot: int) -> tuple:
        return tuple(int(x) for x in self._read(lits=True)[0][slot])

    def literal_columns(self) -> list:
        lits = self._read(lits=True)[0]
        return [lits[:, j].copy() for j in range(self.size)]


class DeviceClauseStore:
    """The clause store as seen from the host (engine.py:203-235)."""

    def __init__(self, engine: "Engine"):
        self._e = engine

    def __len__(self) -> int:
        n = C.c_int64(0)
        check(self._e._L.tsg_store_size(self._e._h, C.byref(n)))
        return n.value

    @property
    def buckets(self) -> Dict[int, BucketView]:
        """Size -> bucket, in creation order (dict insertion order)."""
        nb = C.c_int32(0)
        check(self._e._L.tsg_bucket_count(self._e._h, C.byref(nb)))
        out = {}
        for b in range(nb.value):
            s = C.c_int32(0)
            n = C.c_int64(0)
            check(self._e._L.tsg_bucket_info(self._e._h, b, C.byref(s), C.byref(n)))
            out[s.value] = BucketView(self._e, b, s.value)
        return out

    def clauses(self):
        """(engine_id, lits, origin, activity), sorted by size then slot (engine.py:221-231)."""
        for size, bv in sorted(self.buckets.items()):
            lits, ids, org, acts = bv._read(True, True, True, True)
            for k in range(len(ids)):
                yield int(ids[k]), tuple(int(x) for x in lits[k]), int(org[k]), float(acts[k])

    def scale_activities(self, factor: float) -> None:
        check(self._e._L.tsg_scale_activities(self._e._h, factor))


class Engine:
    """Owns the HBM clause store and runs the exchange rounds on the GPU."""

    def __init__(self, num_vars: int, thread_count: int, config: Optional[EngineConfig] = None):
        self.config = config or EngineConfig()
        self.num_vars = num_vars
        self.thread_count = thread_count
        self._L = _lib.load()
        cfg = _lib.tsg_config(self.config.lane_width, self.config.group_width, self.config.device,
                              _lib.TSG_F_TIMING if self.config.timing else 0,
                              self.config.report_capacity)
        h = C.c_void_p()
        check(self._L.tsg_create(num_vars, C.byref(cfg), C.byref(h)))
        self._h = h
        w = C.c_int64(0)
        check(self._L.tsg_packed_words(num_vars, C.byref(w)))
        self._packed_words = w.value
        self._rec_dtype = REPORT_DTYPE
        self._rec_bytes = 16
        if self.config.lane_width <= 32:  # 12-byte egress records: a quarter fewer bytes D2H
            check(self._L.tsg_set_record_bytes(self._h, 12))
            self._rec_dtype = _reports.RECORD12_DTYPE
            self._rec_bytes = 12
        self.store = DeviceClauseStore(self)
        self._lits: Dict[int, tuple] = {}
        self._size_rank: Dict[int, int] = {}
        self._rank_of_size = np.zeros(64, dtype=np.int64)   # bucket creation rank by clause size
        self._size_of = np.zeros(1024, dtype=np.int32)      # clause size by engine id

        self._id_lock = threading.Lock()
        self._next_id = 0
        self._staged: List[Tuple[int, tuple, int]] = []

        self._queue_lock = threading.Lock()
        self._snapshots: Dict[int, deque] = {t: deque() for t in range(thread_count)}
        self._reports: Dict[int, deque] = {t: deque() for t in range(thread_count)}
        self._pending_reports: Dict[int, int] = {}

        self._activity_inc = 1.0
        self._reduce_watermark = 0
        self.last_round: Optional[_lib.tsg_round_result] = None

        self.counters = {
            "rounds": 0, "clauses_added": 0, "clauses_dropped": 0, "clauses_removed": 0,
            "reduces": 0, "snapshots_accepted": 0, "snapshots_dropped": 0,
            "snapshots_consumed": 0, "aggregate_tests": 0, "aggregate_tests_negative": 0,
            "lane_tests": 0, "lane_triggers": 0, "reports_delivered": 0, "busy_seconds": 0.0,
        }
        self.trace: List[RoundTrace] = []

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.tsg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------
    # producer side (solver threads), engine.py:305-343

    def add_clause(self, lits: Sequence[int], origin: int) -> int:
        lits = tuple(lits)
        with self._id_lock:
            engine_id = self._next_id
            self._next_id += 1
            self._staged.append((engine_id, lits, origin))
        return engine_id

    def submit_assignment(self, snapshot) -> bool:
        """engine.py:319-333.  The snapshot is packed to 2 bits per variable
        here, in the submitting solver thread (tsg_pack_rows releases the GIL),
        where the reference keeps the int8 array; a wrong length is reported
        by run_round, as in the reference (bitpack.py:92-103)."""
        cap = self.config.assignment_queue_capacity
        with self._queue_lock:
            q = self._snapshots.setdefault(snapshot.thread_id, deque())
            if len(q) >= cap:
                self.counters["snapshots_dropped"] += 1
                return False
        packed = self._pack(snapshot.values)
        with self._queue_lock:
            q = self._snapshots.setdefault(snapshot.thread_id, deque())
            if len(q) >= cap:  # filled up while this thread was packing
                self.counters["snapshots_dropped"] += 1
                return False
            q.append((snapshot, packed))
            self.counters["snapshots_accepted"] += 1
            return True

    def _pack(self, values):
        vals = np.ascontiguousarray(np.asarray(values, dtype=np.int8))
        if vals.ndim != 1 or vals.shape[0] != self.num_vars + 1:
            return vals.shape[0] if vals.ndim == 1 else -1  # length error, raised by run_round
        out = np.empty((1, self._packed_words), dtype=np.uint64)
        check(self._L.tsg_pack_rows(ptr(vals), 1, vals.shape[0], self.num_vars, ptr(out), self._packed_words))
        return out

    def drain_reports(self, thread_id: int) -> List[Report]:
        """engine.py:335-343.  A round queues each destination's reports as
        one batch (literals captured at round time); the Report objects are
        built here, in the draining solver thread, off the engine worker."""
        with self._queue_lock:
            q = self._reports.get(thread_id)
            if not q:
                return []
            items = list(q)
            q.clear()
            self._pending_reports[thread_id] = 0
        out: List[Report] = []
        for it in items:
            if isinstance(it, _ReportBatch):
                out.extend(map(Report, itertools.repeat(thread_id, len(it.eids)), it.lits, it.eids, it.masks))
            else:
                out.append(it)
        return out

    # ------------------------------------------------------------------
    # engine worker side

    def _insert(self, batch) -> None:
        """Append staged (id, lits, origin) to the device store at the current
        activity increment (engine.py:357)."""
        if not batch:
            return
        n = len(batch)
        lens = np.fromiter((len(b[1]) for b in batch), dtype=np.int64, count=n)
        offs = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=offs[1:])
        total = int(offs[-1])
        flat = np.fromiter(itertools.chain.from_iterable(b[1] for b in batch), dtype=np.int32, count=total) \
            if total else np.zeros(1, dtype=np.int32)
        ids = np.fromiter((b[0] for b in batch), dtype=np.int64, count=n)
        org = np.fromiter((b[2] for b in batch), dtype=np.int32, count=n)
        check(self._L.tsg_add_clauses(self._h, ptr(flat), ptr(offs), n, ptr(ids), ptr(org),
                                      self._activity_inc))
        self._lits.update((b[0], b[1]) for b in batch)
        # bucket creation order (dict insertion order): new sizes in first-seen order
        sizes, first = np.unique(lens, return_index=True)
        for size in sizes[np.argsort(first, kind="stable")].tolist():
            if size not in self._size_rank:
                self._size_rank[size] = len(self._size_rank)
                if size >= len(self._rank_of_size):
                    grown = np.zeros(max(size + 1, 2 * len(self._rank_of_size)), dtype=np.int64)
                    grown[:len(self._rank_of_size)] = self._rank_of_size
                    self._rank_of_size = grown
                self._rank_of_size[size] = self._size_rank[size]
        top = int(ids.max()) + 1
        if top > len(self._size_of):
            grown = np.zeros(max(top, 2 * len(self._size_of)), dtype=np.int32)
            grown[:len(self._size_of)] = self._size_of
            self._size_of = grown
        self._size_of[ids] = lens
        self.counters["clauses_added"] += n

    def _integrate_exports(self) -> None:
        """engine.py:348-358, batched: insert while there is room; when full,
        reduce once per incoming clause and drop it if still full."""
        with self._id_lock:
            staged, self._staged = self._staged, []
        i, n = 0, len(staged)
        size = len(self.store)
        while i < n:
            room = self.config.max_clauses - size
            if room > 0:
                take = staged[i:i + room]
                self._insert(take)
                size += len(take)
                i += len(take)
                continue
            self.reduce_store()
            size = len(self.store)
            if size >= self.config.max_clauses:
                self.counters["clauses_dropped"] += 1
                i += 1

    def _drain_snapshots(self) -> Dict[int, list]:
        with self._queue_lock:
            pending = {}
            for tid, q in self._snapshots.items():
                if q:
                    pending[tid] = list(q)
                    q.clear()
            return pending

    def run_round(self) -> RoundResult:
        """engine.py:369-435 with the test phase on the GPU."""
        started = time.perf_counter()
        self._integrate_exports()
        store_snapshot = None
        if self.config.trace:
            store_snapshot = [(eid, lits) for eid, lits, _, _ in self.store.clauses()]
        pending = self._drain_snapshots()
        result = RoundResult()
        result.assignments_consumed = sum(len(v) for v in pending.values())
        self.counters["snapshots_consumed"] += result.assignments_consumed

        # grouping (engine.py:390-399): tids ascending, lane_width per group
        lane_width = self.config.lane_width
        rows, lanes, tids = [], [], []
        for tid in sorted(pending):
            snaps = pending[tid]
            for i in range(0, len(snaps), lane_width):
                chunk = snaps[i:i + lane_width]
                for j, (_, packed) in enumerate(chunk):
                    if not isinstance(packed, np.ndarray):
                        raise ValueError(f"assignment {j} has {packed} slots, expected {self.num_vars + 1}")
                    rows.append(packed)
                lanes.append(len(chunk))
                tids.append(tid)

        n_rep = 0
        if lanes:
            block = np.concatenate(rows)
            check(self._L.tsg_stage_packed(self._h, ptr(block), block.shape[0], block.shape[1], 0))
            gl = np.asarray(lanes, dtype=np.int32)
            gt = np.asarray(tids, dtype=np.int32)
            if self.config.lane_width <= 32:
                # 8-byte records written by the kernel when ids and groups fit,
                # else the 12-byte form (include/tsg.h tsg_set_record_bytes)
                nb = 8 if (self._next_id <= (1 << 27) and len(lanes) <= 32) else 12
                if nb != self._rec_bytes:
                    check(self._L.tsg_set_record_bytes(self._h, nb))
                    self._rec_bytes = nb
                    self._rec_dtype = _reports.RECORD8_DTYPE if nb == 8 else _reports.RECORD12_DTYPE
            res = _lib.tsg_round_result()
            check(self._L.tsg_round(self._h, ptr(gl), ptr(gt), len(lanes), self._activity_inc, C.byref(res)))
            self.last_round = res
            self.counters["aggregate_tests"] += res.aggregate_tests
            self.counters["lane_tests"] += res.lane_tests
            self.counters["lane_triggers"] += res.lane_triggers
            self.counters["aggregate_tests_negative"] += res.aggregate_tests_negative
            result.clauses_tested = res.clauses_tested
            result.aggregate_tests_negative = res.aggregate_tests_negative
            recs = _reports.decode(self._fetch(res.reports))
            if len(recs):
                brank = self._rank_of_size[self._size_of[recs["engine_id"]]]
                recs = recs[_reports.reference_order(recs, self.config.group_width, brank)]
                dest = np.asarray(tids, dtype=np.int64)[recs["group"]]
                order = np.argsort(dest, kind="stable")  # per destination, in emission order
                eids = recs["engine_id"][order].tolist()
                lits_of = self._lits
                lits = [lits_of[e] for e in eids]  # captured now: a later reduce may drop the clause
                masks = recs["lane_mask"][order].tolist()
                dsorted = dest[order]
                cuts = np.flatnonzero(np.diff(dsorted)) + 1
                bounds = [0] + cuts.tolist() + [len(eids)]
                batches = [(int(dsorted[a]), _ReportBatch(lits[a:b], eids[a:b], masks[a:b]))
                           for a, b in zip(bounds[:-1], bounds[1:])]
                n_rep = len(eids)
                if self.config.trace:  # the trace keeps Report objects in emission order
                    emitted = [None] * n_rep
                    for k, i in enumerate(order.tolist()):
                        emitted[i] = Report(int(dsorted[k]), lits[k], eids[k], masks[k])

        if n_rep:
            with self._queue_lock:
                for d, batch in batches:
                    self._reports.setdefault(d, deque()).append(batch)
                    self._pending_reports[d] = self._pending_reports.get(d, 0) + len(batch.eids)
            self.counters["reports_delivered"] += n_rep
            result.reports_emitted = n_rep

        if result.assignments_consumed:  # engine.py:416-420
            self._activity_inc /= self.config.activity_decay
            if self._activity_inc > _ACTIVITY_RESCALE:
                self.store.scale_activities(1.0 / _ACTIVITY_RESCALE)
                self._activity_inc /= _ACTIVITY_RESCALE

        if len(self.store) > self.config.max_clauses:
            self.reduce_store()

        if self.config.trace:
            self.trace.append(RoundTrace(
                snapshots=[(s.thread_id, np.array(s.values, copy=True))
                           for snaps in pending.values() for s, _ in snaps],
                store=store_snapshot, reports=emitted if n_rep else []))

        self.counters["rounds"] += 1
        self.counters["busy_seconds"] += time.perf_counter() - started
        return result

    def _fetch(self, n: int) -> np.ndarray:
        recs = np.zeros(n, dtype=self._rec_dtype)
        if n:
            got = C.c_int64(0)
            check(self._L.tsg_fetch_reports(self._h, ptr(recs), n, C.byref(got)))
            recs = recs[:got.value]
        return recs

    def reduce_store(self) -> int:
        """engine.py:469-505; selection and compaction run on the GPU."""
        total = len(self.store)
        if total == 0:
            self._reduce_watermark = self._next_id
            return 0
        target = int(total * (1.0 - self.config.reduce_keep_fraction))
        removed = C.c_int64(0)
        ids = np.zeros(max(target, 1), dtype=np.int64)
        check(self._L.tsg_reduce(self._h, self._reduce_watermark, target, C.byref(removed), ptr(ids)))
        for eid in ids[:removed.value].tolist():
            self._lits.pop(eid, None)
        with self._id_lock:
            self._reduce_watermark = self._next_id
        self.counters["reduces"] += 1
        self.counters["clauses_removed"] += removed.value
        return removed.value

    def remove_clauses(self, engine_ids: Sequence[int]) -> int:
        """Explicit deletion (streaming config C4); order-preserving like
        _SizeBucket.compact (engine.py:184-200).  Ids still staged (added since
        the last round) or already gone are ignored."""
        ids = np.asarray(list(engine_ids), dtype=np.int64)
        if ids.size == 0:
            return 0
        removed = C.c_int64(0)
        check(self._L.tsg_remove_clauses(self._h, ptr(ids), ids.size, C.byref(removed)))
        for eid in ids.tolist():
            self._lits.pop(eid, None)
        self.counters["clauses_deleted"] = self.counters.get("clauses_deleted", 0) + removed.value
        return removed.value

    def serve(self, stop: threading.Event, idle_sleep: float = 0.0005) -> None:
        while not stop.is_set():
            result = self.run_round()
            if result.assignments_consumed == 0:
                time.sleep(idle_sleep)

    def raw_counters(self) -> dict:
        out = dict(self.counters)
        out["store_size"] = len(self.store)
        with self._id_lock:
            out["staged_pending"] = len(self._staged)
        with self._queue_lock:
            out["reports_pending"] = sum(self._pending_reports.values())
            out["snapshots_pending"] = sum(len(q) for q in self._snapshots.values())
        return out
