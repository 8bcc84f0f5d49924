"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  The product package
(paper_2012_03119_b200) never imports it: the product has no CPU path.

`OracleEngine` restates the reference Engine's host logic
(/root/reference/pkg/src/triggersat/engine.py:257-525) on top of the C
restatement in tsg_oracle.c, so a scenario can be replayed against it and
compared with the golden fixtures produced by the reference itself.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from collections import deque
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtsg_oracle.so")

_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


class ora_report(C.Structure):
    _fields_ = [("engine_id", C.c_int64), ("lane_mask", C.c_uint64), ("group", C.c_int32),
                ("bucket", C.c_int32), ("slot", C.c_int64)]


class ora_counters(C.Structure):
    _fields_ = [("clauses_tested", C.c_int64), ("aggregate_tests", C.c_int64),
                ("aggregate_tests_negative", C.c_int64), ("lane_tests", C.c_int64),
                ("lane_triggers", C.c_int64), ("reports", C.c_int64)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.ora_pack.argtypes = [P, C.c_int64, C.c_int64, C.c_int32, C.c_int32, P, P, P]
        L.ora_aggregate.argtypes = [P, P, P, C.c_int32, C.c_int32, C.c_int32, P, P, P]
        L.ora_assignment_trigger.argtypes = [P, P, C.c_int32, C.c_uint64, P, C.c_int32]
        L.ora_assignment_trigger.restype = C.c_uint64
        L.ora_aggregate_trigger.argtypes = [P, P, P, C.c_int32, C.c_int32, P, C.c_int32]
        L.ora_aggregate_trigger.restype = C.c_uint64
        L.ora_store_new.restype = P
        L.ora_store_free.argtypes = [P]
        L.ora_store_insert.argtypes = [P, P, C.c_int32, C.c_int64, C.c_int32, C.c_double]
        L.ora_store_insert_many.argtypes = [P, P, P, C.c_int64, P, P, C.c_double]
        L.ora_store_size.argtypes = [P]
        L.ora_store_size.restype = C.c_int64
        L.ora_store_nbuckets.argtypes = [P]
        L.ora_store_bucket_info.argtypes = [P, C.c_int32, P, P]
        L.ora_store_bucket_read.argtypes = [P, C.c_int32, P, P, P, P]
        L.ora_store_scale.argtypes = [P, C.c_double]
        L.ora_store_reduce.argtypes = [P, C.c_int64, C.c_int64, P]
        L.ora_store_reduce.restype = C.c_int64
        L.ora_store_remove.argtypes = [P, P, C.c_int64]
        L.ora_store_remove.restype = C.c_int64
        L.ora_test_round.argtypes = [P, C.c_int32, P, C.c_int64, P, P, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_double, C.c_int32, C.POINTER(C.POINTER(ora_report)),
                                     C.POINTER(C.c_int64), C.POINTER(ora_counters)]
        L.ora_free.argtypes = [P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# bitpack restatement

def pack(assignments: Sequence[Sequence[int]], num_vars: int, lane_width: int = 32):
    """bitpack.py:81-117 -> (is_true u64[V+1], is_set u64[V+1], lane_mask)."""
    n = len(assignments)
    vals = np.zeros((max(n, 1), num_vars + 1), dtype=np.int8)
    for i, a in enumerate(assignments):
        vals[i] = np.asarray(a, dtype=np.int8)
    t = np.zeros(num_vars + 1, dtype=np.uint64)
    s = np.zeros(num_vars + 1, dtype=np.uint64)
    m = np.zeros(1, dtype=np.uint64)
    rc = lib().ora_pack(_p(vals), n, num_vars + 1, num_vars, lane_width, _p(t), _p(s), _p(m))
    if rc == -1:
        raise ValueError("lane_width out of range")
    if rc == -2:
        raise ValueError("capacity")
    return t, s, int(m[0])


def aggregate(packed: List[Tuple[np.ndarray, np.ndarray]], lane_counts: Sequence[int],
              num_vars: int, group_width: int):
    """bitpack.py:152-167,211-244 -> (cbt, cbf, cbu) u64[V+1]."""
    g = len(packed)
    T = np.zeros((max(g, 1), num_vars + 1), dtype=np.uint64)
    S = np.zeros((max(g, 1), num_vars + 1), dtype=np.uint64)
    for i, (t, s) in enumerate(packed):
        T[i], S[i] = t, s
    lc = np.asarray(list(lane_counts) or [0], dtype=np.int32)
    out = np.zeros((3, num_vars + 1), dtype=np.uint64)
    rc = lib().ora_aggregate(_p(T), _p(S), _p(lc), g, num_vars, group_width,
                             _p(out[0]), _p(out[1]), _p(out[2]))
    if rc:
        raise ValueError("aggregate width/capacity")
    return out[0], out[1], out[2]


def assignment_trigger(is_true, is_set, lane_width, lane_mask, clause) -> int:
    lits = np.asarray(list(clause) or [0], dtype=np.int32)
    return int(lib().ora_assignment_trigger(_p(is_true), _p(is_set), lane_width,
                                             C.c_uint64(lane_mask), _p(lits), len(clause)))


def aggregate_trigger(cbt, cbf, cbu, group_width, group_count, clause) -> int:
    lits = np.asarray(list(clause) or [0], dtype=np.int32)
    return int(lib().ora_aggregate_trigger(_p(cbt), _p(cbf), _p(cbu), group_width, group_count,
                                            _p(lits), len(clause)))


# ---------------------------------------------------------------------------
# store + round restatement

class OracleStore:
    def __init__(self):
        self.h = lib().ora_store_new()

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_store_free(self.h)
            self.h = None

    def insert(self, lits, engine_id, origin, activity):
        a = np.asarray(list(lits) or [0], dtype=np.int32)
        lib().ora_store_insert(self.h, _p(a), len(lits), engine_id, origin, activity)

    def insert_many(self, clauses, ids, origins, activity):
        for c, i, o in zip(clauses, ids, origins):
            self.insert(c, int(i), int(o), activity)

    def insert_flat(self, flat, offsets, ids, origins=None, activity=1.0):
        flat = np.ascontiguousarray(flat, np.int32)
        if flat.size == 0:
            flat = np.zeros(1, np.int32)
        offsets = np.ascontiguousarray(offsets, np.int64)
        ids = np.ascontiguousarray(ids, np.int64)
        org = None if origins is None else np.ascontiguousarray(origins, np.int32)
        lib().ora_store_insert_many(self.h, _p(flat), _p(offsets), len(offsets) - 1, _p(ids),
                                    _p(org) if org is not None else None, activity)

    def __len__(self):
        return int(lib().ora_store_size(self.h))

    def buckets(self):
        """[(size, count, lits[count,size], ids, origins, acts)] in creation order."""
        out = []
        for b in range(lib().ora_store_nbuckets(self.h)):
            size = np.zeros(1, np.int32)
            cnt = np.zeros(1, np.int64)
            lib().ora_store_bucket_info(self.h, b, _p(size), _p(cnt))
            s, n = int(size[0]), int(cnt[0])
            lits = np.zeros((n, s), np.int32)
            ids = np.zeros(n, np.int64)
            org = np.zeros(n, np.int32)
            acts = np.zeros(n, np.float64)
            lib().ora_store_bucket_read(self.h, b, _p(lits), _p(ids), _p(org), _p(acts))
            out.append((s, n, lits, ids, org, acts))
        return out

    def clauses(self):
        """engine.py:221-231 order: sorted by size, then slot."""
        for s, n, lits, ids, org, acts in sorted(self.buckets(), key=lambda b: b[0]):
            for k in range(n):
                yield int(ids[k]), tuple(int(x) for x in lits[k]), int(org[k]), float(acts[k])

    def scale(self, f):
        lib().ora_store_scale(self.h, f)

    def reduce(self, eligible_below, target):
        out = np.zeros(max(target, 1), np.int64)
        n = lib().ora_store_reduce(self.h, eligible_below, target, _p(out))
        return int(n), out[:n]

    def remove(self, ids):
        a = np.asarray(list(ids) or [0], np.int64)
        return int(lib().ora_store_remove(self.h, _p(a), len(ids)))

    def test_round(self, num_vars, snaps: np.ndarray, group_lanes, group_tid, lane_width,
                   group_width, activity_inc, nthreads=1):
        snaps = np.ascontiguousarray(snaps, dtype=np.int8)
        if snaps.ndim != 2:
            snaps = snaps.reshape(-1, num_vars + 1)
        gl = np.asarray(group_lanes, np.int32)
        gt = np.asarray(group_tid, np.int32)
        outp = C.POINTER(ora_report)()
        n = C.c_int64(0)
        ctr = ora_counters()
        rc = lib().ora_test_round(self.h, num_vars, _p(snaps) if snaps.size else None,
                                  snaps.shape[1] if snaps.size else num_vars + 1,
                                  _p(gl) if gl.size else None, _p(gt) if gt.size else None,
                                  len(gl), lane_width, group_width, activity_inc, nthreads,
                                  C.byref(outp), C.byref(n), C.byref(ctr))
        if rc:
            raise ValueError(f"ora_test_round rc={rc}")
        recs = np.ctypeslib.as_array(outp, shape=(n.value,)).copy() if n.value else \
            np.zeros(0, dtype=np.dtype([("engine_id", "<i8"), ("lane_mask", "<u8"), ("group", "<i4"),
                                        ("bucket", "<i4"), ("slot", "<i8")]))
        lib().ora_free(C.cast(outp, C.c_void_p))
        counters = {k: getattr(ctr, k) for k, _ in ora_counters._fields_}
        return recs, counters


# ---------------------------------------------------------------------------
# engine restatement (host logic of engine.py:257-525 over the C oracle)

@dataclass
class OReport:
    destination: int
    lits: tuple
    engine_id: int
    lane_mask: int


class OracleEngine:
    ACTIVITY_RESCALE = 1e100

    def __init__(self, num_vars, thread_count, max_clauses=5_000_000, assignment_queue_capacity=None,
                 lane_width=32, group_width=32, activity_decay=0.999, reduce_keep_fraction=0.5,
                 nthreads=1, **_ignored):
        self.num_vars = num_vars
        self.max_clauses = max_clauses
        self.cap = assignment_queue_capacity if assignment_queue_capacity is not None else 2 * lane_width
        self.lane_width, self.group_width = lane_width, group_width
        self.decay, self.keep = activity_decay, reduce_keep_fraction
        self.nthreads = nthreads
        self.store = OracleStore()
        self.lits: Dict[int, tuple] = {}
        self.next_id = 0
        self.staged: List[Tuple[int, tuple, int]] = []
        self.snaps: Dict[int, deque] = {t: deque() for t in range(thread_count)}
        self.reports: Dict[int, deque] = {t: deque() for t in range(thread_count)}
        self.inc = 1.0
        self.watermark = 0
        self.counters = dict(rounds=0, clauses_added=0, clauses_dropped=0, clauses_removed=0, reduces=0,
                             snapshots_accepted=0, snapshots_dropped=0, snapshots_consumed=0,
                             aggregate_tests=0, aggregate_tests_negative=0, lane_tests=0,
                             lane_triggers=0, reports_delivered=0)
        self._lock = threading.Lock()

    def add_clause(self, lits, origin):  # engine.py:305-317
        eid = self.next_id
        self.next_id += 1
        self.staged.append((eid, tuple(lits), origin))
        return eid

    def submit_assignment(self, tid, values, seq=0):  # engine.py:319-333
        q = self.snaps.setdefault(tid, deque())
        if len(q) >= self.cap:
            self.counters["snapshots_dropped"] += 1
            return False
        q.append(np.asarray(values, dtype=np.int8))
        self.counters["snapshots_accepted"] += 1
        return True

    def drain_reports(self, tid):  # engine.py:335-343
        q = self.reports.get(tid)
        if not q:
            return []
        out = list(q)
        q.clear()
        return out

    def remove_clauses(self, ids):  # explicit delete (C4): _SizeBucket.compact with a keep mask
        ids = [int(i) for i in ids]
        removed = self.store.remove(ids)
        for i in ids:
            self.lits.pop(i, None)
        return removed

    def reduce_store(self):  # engine.py:469-505
        total = len(self.store)
        if total == 0:
            self.watermark = self.next_id
            return 0
        target = int(total * (1.0 - self.keep))
        removed, ids = self.store.reduce(self.watermark, target)
        for i in ids:
            self.lits.pop(int(i), None)
        self.watermark = self.next_id
        self.counters["reduces"] += 1
        self.counters["clauses_removed"] += removed
        return removed

    def run_round(self):  # engine.py:369-435
        staged, self.staged = self.staged, []
        for eid, lits, origin in staged:
            if len(self.store) >= self.max_clauses:
                self.reduce_store()
                if len(self.store) >= self.max_clauses:
                    self.counters["clauses_dropped"] += 1
                    continue
            self.store.insert(lits, eid, origin, self.inc)
            self.lits[eid] = lits
            self.counters["clauses_added"] += 1
        pending = {t: list(q) for t, q in self.snaps.items() if q}
        for q in self.snaps.values():
            q.clear()
        consumed = sum(len(v) for v in pending.values())
        self.counters["snapshots_consumed"] += consumed
        rows, lanes, tids = [], [], []
        for tid in sorted(pending):
            s = pending[tid]
            for i in range(0, len(s), self.lane_width):
                chunk = s[i:i + self.lane_width]
                rows.extend(chunk)
                lanes.append(len(chunk))
                tids.append(tid)
        result = dict(reports_emitted=0, clauses_tested=0, assignments_consumed=consumed,
                      aggregate_tests_negative=0)
        if lanes:
            snaps = np.stack(rows).astype(np.int8)
            recs, ctr = self.store.test_round(self.num_vars, snaps, lanes, tids, self.lane_width,
                                              self.group_width, self.inc, self.nthreads)
            for k in ("aggregate_tests", "aggregate_tests_negative", "lane_tests", "lane_triggers"):
                self.counters[k] += ctr[k]
            result["clauses_tested"] = ctr["clauses_tested"]
            result["aggregate_tests_negative"] = ctr["aggregate_tests_negative"]
            for r in recs:
                tid = tids[int(r["group"])]
                eid = int(r["engine_id"])
                self.reports.setdefault(tid, deque()).append(
                    OReport(tid, self.lits[eid], eid, int(r["lane_mask"])))
            self.counters["reports_delivered"] += len(recs)
            result["reports_emitted"] = len(recs)
        if consumed:
            self.inc /= self.decay
            if self.inc > self.ACTIVITY_RESCALE:
                self.store.scale(1.0 / self.ACTIVITY_RESCALE)
                self.inc /= self.ACTIVITY_RESCALE
        if len(self.store) > self.max_clauses:
            self.reduce_store()
        self.counters["rounds"] += 1
        return result
