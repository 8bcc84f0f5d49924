"""The clause-exchange engine on B200s: drop-in for triggersat.engine.Engine.

Same public surface as the reference (engine.py:44-525): ``EngineConfig``,
``AssignmentSnapshot``, ``Report``, ``RoundResult``, ``RoundTrace`` and
``Engine`` with ``add_clause`` / ``submit_assignment`` / ``drain_reports`` /
``run_round`` / ``reduce_store`` / ``serve`` / ``raw_counters`` / ``store`` /
``counters`` / ``trace`` / ``config``.  The host keeps what the reference
keeps on its producer side -- the id lock, the staging list, the per-thread
snapshot and report queues (engine.py:273-279) -- and the clause store lives
in HBM behind the C ABI (include/tsg.h): size buckets, activities, ids and
the round's kernels.

Host data paths, none of them per-record Python work:

* snapshots are packed (2 bits per variable, tsg_pack_rows, GIL released)
  by the submitting solver thread into that thread's page-locked queue
  region and copied to the device at once (tsg_ingress_copy, the engine's
  ingress stream); a round stages every thread's device region as one
  segment (tsg_stage_packed_segments) -- no host copy of the rows and no
  host-to-device copy on the round's path;
* a round's reports are ordered on the GPU into the reference's delivery
  order (tsg_fetch_ordered) and queued per destination as array slices;
  the ``Report`` objects, with their literals from a literal
  arena, are built by the draining solver thread;
* ``EngineConfig.devices`` names several GPUs: the clauses are sharded
  across them (every size bucket balanced), the round's tables are encoded
  once and copied peer to peer (tsg_round_tables_copy, NVLink), every GPU
  tests its shard, and the records of all shards are ordered together;
  ``reduce_store`` stays exact (sharded.global_reduce).

There is no CPU path: constructing an Engine without the CUDA library or a
CUDA device raises.
"""
from __future__ import annotations

import array
import ctypes as C
import threading
import time
from collections import deque
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from . import reports as _reports
from . import sharded as _sharded
from ._lib import check, ptr
from .native import NativeEngine, RingDrainer

#: Activities are rescaled when the bump increment passes this (engine.py:39-40).
_ACTIVITY_RESCALE = 1e100


@dataclass
class EngineConfig:
    """Tunables, identical to the reference (engine.py:44-74) plus the device
    ordinal(s) and the initial report-buffer size."""

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
    devices: Optional[Sequence[int]] = None  # clause shards, one engine per entry (default: [device])
    chunk_filter: bool = False  # multi-chunk rounds: chunk-level aggregate sweep first
    # > 0: the rounds' records go through a page-locked host ring of this many
    # records, drained by CPU threads while the kernel runs (tsg_ring_*,
    # DESIGN.md §4.4), and are put in delivery order on the host -- for rounds
    # with few reports; 0: device record buffer, ordered on the GPU
    report_ring: int = 0

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
        if self.devices is not None and len(self.devices) < 1:
            raise ValueError("devices must name at least one GPU")
        if self.report_ring < 0:
            raise ValueError("report_ring must be >= 0")
        if self.report_ring and self.lane_width > 32:
            raise ValueError("report_ring carries 32-bit lane masks: lane_width must be <= 32")


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
    """One round's reports for one destination, in delivery order: engine
    ids and lane masks (views of the round's page-locked record buffer,
    `keep`), with the literal arena as it was at round time."""

    eids: np.ndarray
    masks: np.ndarray
    arena: "_Arena"
    keep: object = None

    def __len__(self):
        return len(self.eids)


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


class _Arena:
    """Literal arena by engine id (Report.lits, engine.py:90-102).  Arrays
    are never rewritten in place where a report batch may read them: appends
    write past `used` and set the entries of new ids only, and reclaiming the
    literals of removed clauses (once they outweigh the live ones) builds
    new arrays -- a batch holding the arena of its round keeps valid
    literals even after its clause was removed."""

    __slots__ = ("lits", "off", "size", "used", "alive", "live_lits", "dead_lits")
    RECLAIM_MIN = 1 << 20  # dead literals below this are never worth a rebuild

    def __init__(self, lits=None, off=None, size=None, used=0):
        self.lits = np.zeros(1024, np.int32) if lits is None else lits
        self.off = np.zeros(1024, np.int64) if off is None else off
        self.size = np.zeros(1024, np.int32) if size is None else size
        self.used = used
        self.alive = np.zeros(self.off.size, bool)  # (the live arena only; snapshots do not use it)
        self.live_lits = 0
        self.dead_lits = 0

    def snapshot(self) -> "_Arena":
        """A read-only view for a report batch (lits_of only)."""
        v = object.__new__(_Arena)
        v.lits, v.off, v.size, v.used = self.lits, self.off, self.size, self.used
        v.alive, v.live_lits, v.dead_lits = None, 0, 0
        return v

    def append(self, ids: np.ndarray, lens: np.ndarray, flat: np.ndarray) -> None:
        total = int(flat.size)
        if self.used + total > self.lits.size:  # grow by half again (no zero fill: only [0, used) is read)
            grown = np.empty(max(self.used + total, self.lits.size + self.lits.size // 2), np.int32)
            grown[:self.used] = self.lits[:self.used]
            self.lits = grown
        self.lits[self.used:self.used + total] = flat
        top = int(ids.max()) + 1 if ids.size else 0
        if top > self.off.size:
            n = max(top, self.off.size + self.off.size // 2)
            off = np.zeros(n, np.int64)
            off[:self.off.size] = self.off
            size = np.zeros(n, np.int32)
            size[:self.size.size] = self.size
            alive = np.zeros(n, bool)
            alive[:self.alive.size] = self.alive
            self.off, self.size, self.alive = off, size, alive
        starts = np.zeros(len(lens), np.int64)
        if len(lens) > 1:
            np.cumsum(lens[:-1], out=starts[1:])
        if ids.size and int(ids[-1]) - int(ids[0]) == ids.size - 1:  # consecutive ids (the usual batch)
            sl = slice(int(ids[0]), int(ids[-1]) + 1)
            self.off[sl] = self.used + starts
            self.size[sl] = lens
            self.alive[sl] = True
        else:
            self.off[ids] = self.used + starts
            self.size[ids] = lens
            self.alive[ids] = True
        self.used += total
        self.live_lits += total

    def remove(self, ids: np.ndarray) -> None:
        """Clauses gone from the store: their literals are reclaimed once the
        dead outweigh the live (a new set of arrays; report batches keep
        theirs)."""
        ids = np.asarray(ids, np.int64)
        ids = ids[(ids >= 0) & (ids < self.alive.size)]
        ids = np.unique(ids[self.alive[ids]])
        if not ids.size:
            return
        self.alive[ids] = False
        dead = int(self.size[ids].sum())
        self.live_lits -= dead
        self.dead_lits += dead
        if self.dead_lits > max(self.live_lits, self.RECLAIM_MIN):
            self._compact()

    def _compact(self) -> None:
        live = np.nonzero(self.alive)[0]
        sizes = self.size[live].astype(np.int64)
        total = int(sizes.sum())
        starts = np.zeros(live.size, np.int64)
        if live.size > 1:
            np.cumsum(sizes[:-1], out=starts[1:])
        src = np.repeat(self.off[live] - starts, sizes) + np.arange(total, dtype=np.int64)
        lits = np.empty(max(total + total // 2, 1024), np.int32)
        lits[:total] = self.lits[src]
        off = np.zeros(self.off.size, np.int64)
        size = np.zeros(self.size.size, np.int32)
        off[live] = starts
        size[live] = sizes
        self.lits, self.off, self.size, self.used = lits, off, size, total
        self.live_lits, self.dead_lits = total, 0

    def lits_of(self, eid: int) -> tuple:
        o = int(self.off[eid])
        return tuple(self.lits[o:o + int(self.size[eid])].tolist())


class _Run:
    """Clauses staged by consecutive add_clause calls (engine.py:305-317),
    kept flat (C arrays appended under the id lock) so integration needs no
    per-literal Python work."""

    __slots__ = ("first", "lits", "lens", "org")

    def __init__(self, first: int):
        self.first = first
        self.lits = array.array("i")
        self.lens = array.array("i")
        self.org = array.array("i")

    def arrays(self):
        n = len(self.lens)
        return (np.arange(self.first, self.first + n, dtype=np.int64),
                np.frombuffer(self.lens, dtype=np.int32).astype(np.int64) if n else np.zeros(0, np.int64),
                np.frombuffer(self.lits, dtype=np.int32) if len(self.lits) else np.zeros(0, np.int32),
                np.frombuffer(self.org, dtype=np.int32) if n else np.zeros(0, np.int32))


class _PinnedPool:
    """Page-locked host buffers for the rounds' ordered records: the device
    writes them at link rate, and the report batches view them in place.  A
    buffer returns to the pool when the last batch viewing it is drained."""

    class Buf:
        def __init__(self, pool, p, nbytes):
            self.pool, self.p, self.nbytes = pool, p, nbytes

        def __del__(self):
            self.pool._release(self.p, self.nbytes)

    def __init__(self, lib):
        self._lib = lib
        self._lock = threading.Lock()
        self._free: List[Tuple[object, int]] = []
        self._closed = False

    def get(self, nbytes: int) -> "_PinnedPool.Buf":
        with self._lock:
            fit = [f for f in self._free if f[1] >= nbytes]
            if fit:
                f = min(fit, key=lambda x: x[1])
                self._free.remove(f)
                return _PinnedPool.Buf(self, *f)
        size = max(nbytes + nbytes // 2, 1 << 20)
        p = C.c_void_p()
        check(self._lib.tsg_host_alloc(size, C.byref(p)))
        return _PinnedPool.Buf(self, p, size)

    def _release(self, p, nbytes):
        with self._lock:
            if self._closed:
                self._lib.tsg_host_free(p)
            else:
                self._free.append((p, nbytes))

    def close(self):
        with self._lock:
            self._closed = True
            free, self._free = self._free, []
        for p, _ in free:
            self._lib.tsg_host_free(p)


class _SnapQueue:
    """One solver thread's snapshot queue: packed rows in one of two regions
    (the round drains one while submissions fill the other), each a
    page-locked host region plus its device copy -- a submit packs the row
    into host memory and queues its copy to the device on the engine's
    ingress stream (tsg_ingress_copy), so the round finds its rows on the
    device -- plus the snapshot objects for trace mode."""

    def __init__(self, lib, h, cap: int, words: int):
        self.lock = threading.Lock()
        self.cap, self.words = cap, words
        self._lib, self._h = lib, h
        self._raw = [None, None]
        self.dev = [None, None]
        self.rows = [None, None]
        for r in range(2):
            p = C.c_void_p()
            check(lib.tsg_host_alloc(cap * words * 8, C.byref(p)))
            self._raw[r] = p
            self.rows[r] = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint64)), shape=(cap, words))
            d = C.c_void_p()
            check(lib.tsg_device_alloc(h, cap * words * 8, C.byref(d)))
            self.dev[r] = d
        self.cur = 0
        self.n = 0
        self.snaps: List[object] = []
        self.bad: List[int] = []  # lengths of rejected snapshots (raised by run_round)

    def close(self):
        for r in range(2):
            if self._raw[r] is not None:
                self._lib.tsg_host_free(self._raw[r])
                self._raw[r] = None
            if self.dev[r] is not None:
                self._lib.tsg_device_free(self._h, self.dev[r])
                self.dev[r] = None


class _StoreShards:
    """The store as seen from the host: the shards' buckets merged by size,
    slots in engine-id order (engine.py:122-235)."""

    def __init__(self, engine: "Engine"):
        self._e = engine

    def __len__(self) -> int:
        return sum(len(s) for s in self._e._shards)

    @property
    def buckets(self) -> Dict[int, "BucketView"]:
        """Size -> bucket, in creation order (dict insertion order)."""
        return {s: BucketView(self._e, s) for s in self._e._sizes_in_order}

    def clauses(self):
        """(engine_id, lits, origin, activity), sorted by size then slot (engine.py:221-231)."""
        for size in sorted(self._e._sizes_in_order):
            lits, ids, org, acts = BucketView(self._e, size)._read()
            for k in range(len(ids)):
                yield int(ids[k]), tuple(int(x) for x in lits[k]), int(org[k]), float(acts[k])

    def scale_activities(self, factor: float) -> None:
        for s in self._e._shards:
            s.scale(factor)


class BucketView:
    """Live view of one size bucket across the shards (the reference's
    _SizeBucket, engine.py:122-200).  Every attribute read fetches from HBM."""

    def __init__(self, engine: "Engine", size: int):
        self._e, self.size = engine, size

    def _read(self):
        parts = []
        for sh in self._e._shards:
            nb = C.c_int32(0)
            check(sh.L.tsg_bucket_count(sh.h, C.byref(nb)))
            for b in range(nb.value):
                s, n = C.c_int32(0), C.c_int64(0)
                check(sh.L.tsg_bucket_info(sh.h, b, C.byref(s), C.byref(n)))
                if s.value != self.size or not n.value:
                    continue
                out = [np.zeros((n.value, self.size), np.int32), np.zeros(n.value, np.int64),
                       np.zeros(n.value, np.int32), np.zeros(n.value, np.float64)]
                check(sh.L.tsg_bucket_read(sh.h, b, *(ptr(a) for a in out)))
                parts.append(out)
        if not parts:
            return (np.zeros((0, self.size), np.int32), np.zeros(0, np.int64), np.zeros(0, np.int32),
                    np.zeros(0, np.float64))
        lits, ids, org, acts = (np.concatenate([p[i] for p in parts]) for i in range(4))
        o = np.argsort(ids, kind="stable")
        return lits[o], ids[o], org[o], acts[o]

    @property
    def count(self) -> int:
        return len(self._read()[1])

    @property
    def activities(self) -> np.ndarray:
        return self._read()[3]

    @property
    def engine_ids(self) -> np.ndarray:
        return self._read()[1]

    @property
    def origins(self) -> np.ndarray:
        return self._read()[2]

    def lits_at(self, slot: int) -> tuple:
        return tuple(int(x) for x in self._read()[0][slot])

    def literal_columns(self) -> list:
        lits = self._read()[0]
        return [lits[:, j].copy() for j in range(self.size)]


class Engine:
    """Owns the HBM clause store (one shard per configured GPU) and runs the
    exchange rounds on the GPU(s)."""

    def __init__(self, num_vars: int, thread_count: int, config: Optional[EngineConfig] = None):
        self.config = config or EngineConfig()
        self.num_vars = num_vars
        self.thread_count = thread_count
        self._L = _lib.load()
        devices = list(self.config.devices) if self.config.devices else [self.config.device]
        self._shards = [NativeEngine(num_vars, self.config.lane_width, self.config.group_width, device=d,
                                     timing=self.config.timing, report_capacity=self.config.report_capacity,
                                     chunk_filter=self.config.chunk_filter)
                        for d in devices]
        self._h = self._shards[0].h  # the first shard: staging, encode, record ordering
        self._drainers: List[RingDrainer] = []  # report_ring: one drainer thread per shard
        self._shard_reports: List[int] = []     # the last round's records per shard
        if self.config.report_ring:
            for s in self._shards:
                s.ring_open(self.config.report_ring)
                self._drainers.append(RingDrainer(s, threads=1))
        w = C.c_int64(0)
        check(self._L.tsg_packed_words(num_vars, C.byref(w)))
        self._packed_words = w.value
        self._rec_bytes = 16
        self.store = _StoreShards(self)
        self._arena = _Arena()
        self._pinned = _PinnedPool(self._L)
        self._sizes_in_order: List[int] = []                # bucket creation order (dict order)
        self._rank_of_size = np.zeros(64, dtype=np.int32)   # creation rank by clause size
        self._size_known = np.zeros(64, dtype=bool)           # sizes with a bucket
        self._shard_load = np.zeros((len(self._shards), 64), dtype=np.int64)  # clauses per (shard, size)

        self._id_lock = threading.Lock()
        self._next_id = 0
        self._staged: list = []  # _Run (add_clause) and array batches (add_clauses), in id order

        self._queue_lock = threading.Lock()  # report queues, counters, the set of snapshot queues
        self._squeues: Dict[int, _SnapQueue] = {}
        self._reports: Dict[int, deque] = {t: deque() for t in range(thread_count)}
        self._pending_reports: Dict[int, int] = {}

        self._activity_inc = 1.0
        self._reduce_watermark = 0
        self.last_round: Optional[_lib.tsg_round_result] = None
        self.last_phases: Dict[str, float] = {}  # wall ms of the last run_round's phases

        self.counters = {
            "rounds": 0, "clauses_added": 0, "clauses_dropped": 0, "clauses_removed": 0,
            "reduces": 0, "snapshots_accepted": 0, "snapshots_dropped": 0,
            "snapshots_consumed": 0, "aggregate_tests": 0, "aggregate_tests_negative": 0,
            "lane_tests": 0, "lane_triggers": 0, "reports_delivered": 0, "busy_seconds": 0.0,
        }
        self.trace: List[RoundTrace] = []

    def close(self) -> None:
        for d in getattr(self, "_drainers", []):
            d.close()
        for s in getattr(self, "_shards", []) if getattr(self, "_drainers", None) else []:
            s.ring_close()
        self._drainers = []
        for q in getattr(self, "_squeues", {}).values():
            q.close()
        if getattr(self, "_pinned", None) is not None:
            self._pinned.close()
        for s in getattr(self, "_shards", []):
            s.close()
        self._shards = []
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------
    # producer side (solver threads), engine.py:305-343

    def add_clause(self, lits: Sequence[int], origin: int) -> int:
        with self._id_lock:
            engine_id = self._next_id
            self._next_id += 1
            run = self._staged[-1] if self._staged and isinstance(self._staged[-1], _Run) else None
            if run is None:
                run = _Run(engine_id)
                self._staged.append(run)
            n0 = len(run.lits)
            run.lits.extend(lits)
            run.lens.append(len(run.lits) - n0)
            run.org.append(origin)
        return engine_id

    def _queue(self, tid: int) -> _SnapQueue:
        q = self._squeues.get(tid)
        if q is None:
            with self._queue_lock:
                q = self._squeues.get(tid)
                if q is None:
                    q = _SnapQueue(self._L, self._h, self.config.assignment_queue_capacity, self._packed_words)
                    self._squeues[tid] = q
        return q

    def submit_assignment(self, snapshot) -> bool:
        """engine.py:319-333: drop the newest when the thread's queue is full.
        The snapshot is packed into the thread's page-locked queue region
        here, in the submitting solver thread (the reference keeps the int8
        array); a wrong length is reported by run_round, as in the reference
        (bitpack.py:92-103)."""
        q = self._queue(snapshot.thread_id)
        with q.lock:
            if q.n + len(q.bad) >= q.cap:  # (a rejected snapshot still occupies its queue slot)
                ok = False
            else:
                vals = np.ascontiguousarray(np.asarray(snapshot.values, dtype=np.int8))
                if vals.ndim != 1 or vals.shape[0] != self.num_vars + 1:
                    q.bad.append(vals.shape[0] if vals.ndim == 1 else -1)
                else:  # (the GIL is released while the row is packed)
                    off = q.n * q.words * 8
                    host = C.c_void_p(q.rows[q.cur].ctypes.data + off)
                    check(self._L.tsg_pack_rows(ptr(vals), 1, vals.shape[0], self.num_vars, host, q.words))
                    check(self._L.tsg_ingress_copy(self._h, C.c_void_p(q.dev[q.cur].value + off), host, q.words * 8))
                    q.n += 1
                if self.config.trace:
                    q.snaps.append(snapshot)
                ok = True
        with self._queue_lock:
            self.counters["snapshots_accepted" if ok else "snapshots_dropped"] += 1
        return ok

    def drain_reports(self, thread_id: int) -> List[Report]:
        """engine.py:335-343.  A round queues each destination's reports as
        one batch; the Report objects (literals from the arena of that round)
        are built here, in the draining solver thread, off the engine worker."""
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
                ar = it.arena
                offs = ar.off[it.eids].tolist()
                sizes = ar.size[it.eids].tolist()
                lits = ar.lits
                out.extend(Report(thread_id, tuple(lits[o:o + s].tolist()), e, m)
                           for o, s, e, m in zip(offs, sizes, it.eids.tolist(), it.masks.tolist()))
            else:
                out.append(it)
        return out

    # ------------------------------------------------------------------
    # engine worker side

    def add_clauses(self, flat, offsets, origin=0) -> int:
        """Bulk add_clause (an extension of the reference API for loading a
        store): clause i is flat[offsets[i]:offsets[i+1]]; consecutive engine
        ids are assigned under the id lock and the batch is staged like
        add_clause's.  `origin`: one int or one per clause.  Returns the
        first id."""
        flat = np.ascontiguousarray(flat, np.int32)
        offsets = np.ascontiguousarray(offsets, np.int64)
        n = len(offsets) - 1
        org = np.broadcast_to(np.asarray(origin, np.int32), (n,)).copy()
        with self._id_lock:
            first = self._next_id
            self._next_id += n
            self._staged.append((np.arange(first, first + n, dtype=np.int64), np.diff(offsets),
                                 flat[offsets[0]:offsets[-1]], org))
        return first

    def _insert(self, ids: np.ndarray, lens: np.ndarray, flat: np.ndarray, org: np.ndarray) -> None:
        """Append clauses (engine ids ascending) to the store at the current
        activity increment (engine.py:357): shard by size (every bucket
        balanced over the devices), literals into the arena."""
        n = len(ids)
        if not n:
            return
        offs = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=offs[1:])
        # bucket creation order (dict insertion order): new sizes in first-seen
        # order (a batch of known sizes only -- the streaming case -- skips it)
        top = int(lens.max()) + 1
        if top <= self._size_known.size and self._size_known[lens].all():
            sizes = None
        else:
            sizes, first = np.unique(lens, return_index=True)
        if sizes is not None and top > self._rank_of_size.size:
            grown = np.zeros(max(top, 2 * self._rank_of_size.size), np.int32)
            grown[:self._rank_of_size.size] = self._rank_of_size
            self._rank_of_size = grown
            load = np.zeros((len(self._shards), grown.size), np.int64)
            load[:, :self._shard_load.shape[1]] = self._shard_load
            self._shard_load = load
        if sizes is not None:
            known = set(self._sizes_in_order)
            for size in sizes[np.argsort(first, kind="stable")].tolist():
                if size not in known:
                    self._rank_of_size[size] = len(self._sizes_in_order)
                    self._sizes_in_order.append(size)
                    known.add(size)
            self._size_known = np.zeros(self._rank_of_size.size, bool)
            self._size_known[self._sizes_in_order] = True
        ns = len(self._shards)
        if ns == 1:
            self._shards[0].add_clauses(flat, offs, ids, org, self._activity_inc)
        else:  # per size round-robin from each shard's current count: balanced buckets
            order = np.argsort(lens, kind="stable")
            sl = lens[order]
            starts = np.searchsorted(sl, sl, side="left")
            within = np.arange(n) - starts
            base = self._shard_load.sum(axis=0)[sl]
            shard_of = np.empty(n, np.int64)
            shard_of[order] = (base + within) % ns
            for r, sh in enumerate(self._shards):
                sel = np.nonzero(shard_of == r)[0]
                if not sel.size:
                    continue
                so = np.zeros(sel.size + 1, np.int64)
                np.cumsum(lens[sel], out=so[1:])
                keep = np.repeat(shard_of == r, lens)
                sh.add_clauses(flat[keep], so, ids[sel], org[sel], self._activity_inc)
                np.add.at(self._shard_load[r], lens[sel], 1)
        self._arena.append(ids, lens.astype(np.int32), flat)
        self.counters["clauses_added"] += n

    def _integrate_exports(self) -> None:
        """engine.py:348-358, batched: insert while there is room; when full,
        reduce once per incoming clause and drop it if still full."""
        with self._id_lock:
            staged, self._staged = self._staged, []
        if not staged:
            return
        # the staged clauses as arrays, in id order (add_clause runs and add_clauses batches)
        parts = [b.arrays() if isinstance(b, _Run) else b for b in staged]
        ids, lens, flat, org = (np.concatenate([p[k] for p in parts]) for k in range(4))
        offs = np.zeros(len(ids) + 1, dtype=np.int64)
        np.cumsum(lens, out=offs[1:])
        i, n = 0, len(ids)
        size = len(self.store)
        while i < n:
            room = self.config.max_clauses - size
            if room > 0:
                j = min(n, i + room)
                self._insert(ids[i:j], lens[i:j], flat[offs[i]:offs[j]], org[i:j])
                size += j - i
                i = j
                continue
            self.reduce_store()
            size = len(self.store)
            if size >= self.config.max_clauses:
                self.counters["clauses_dropped"] += 1
                i += 1

    def _drain_snapshots(self):
        """Every thread's queued rows, tids ascending: [(tid, rows, n, snaps, bad)];
        each queue switches to its other region for new submissions."""
        with self._queue_lock:
            queues = sorted(self._squeues.items())
        out = []
        for tid, q in queues:
            with q.lock:
                if not q.n and not q.bad:
                    continue
                out.append((tid, q.dev[q.cur].value, q.n, q.snaps, q.bad))
                q.cur ^= 1
                q.n = 0
                q.snaps = []
                q.bad = []
        return out

    def run_round(self) -> RoundResult:
        """engine.py:369-435 with the test phase on the GPU(s)."""
        started = time.perf_counter()
        ph = {}
        self._integrate_exports()
        ph["integrate"] = time.perf_counter()
        store_snapshot = None
        if self.config.trace:
            store_snapshot = [(eid, lits) for eid, lits, _, _ in self.store.clauses()]
        pending = self._drain_snapshots()
        result = RoundResult()
        result.assignments_consumed = sum(n + len(bad) for _, _, n, _, bad in pending)
        self.counters["snapshots_consumed"] += result.assignments_consumed
        for _, _, _, _, bad in pending:
            if bad:  # pack_assignments' length check (bitpack.py:92-103)
                raise ValueError(f"assignment has {bad[0]} slots, expected {self.num_vars + 1}")

        # grouping (engine.py:390-399): tids ascending, lane_width per group
        lw = self.config.lane_width
        lanes, tids = [], []
        for tid, _, n, _, _ in pending:
            for i in range(0, n, lw):
                lanes.append(min(lw, n - i))
                tids.append(tid)
        n_rep = 0
        emitted: list = []
        batches = []
        if lanes:
            gl = np.asarray(lanes, dtype=np.int32)
            gt = np.asarray(tids, dtype=np.int32)
            segs = (C.c_void_p * len(pending))(*[dev for _, dev, _, _, _ in pending])
            cnts = np.asarray([n for _, _, n, _, _ in pending], dtype=np.int64)
            check(self._L.tsg_stage_packed_segments(self._h, segs, ptr(cnts), len(pending), self._packed_words))
            if lw <= 32:
                # 8-byte records written by the kernel when ids and groups fit,
                # else the general 16-byte form (ordered on the device either way)
                nb = 8 if (self._next_id <= (1 << 27) and len(lanes) <= 32) else 16
                if nb != self._rec_bytes:
                    for s in self._shards:
                        s.set_record_bytes(nb)
                    self._rec_bytes = nb
            ph["drain_stage"] = time.perf_counter()
            res = self._round(gl, gt)
            ph["gpu_round"] = time.perf_counter()
            self.last_round = res
            self.counters["aggregate_tests"] += res.aggregate_tests
            self.counters["lane_tests"] += res.lane_tests
            self.counters["lane_triggers"] += res.lane_triggers
            self.counters["aggregate_tests_negative"] += res.aggregate_tests_negative
            result.clauses_tested = res.clauses_tested
            result.aggregate_tests_negative = res.aggregate_tests_negative
            if res.reports:
                dests = [t for t, _, _, _, _ in pending]
                if self._drainers:
                    eids, masks, groups, counts, keep = self._ring_ordered(gt, dests)
                else:
                    eids, masks, groups, counts, keep = self._fetch_ordered(res.reports, len(pending))
                ph["order_fetch"] = time.perf_counter()
                arena = self._arena.snapshot()  # literals as of this round (a later reduce may drop the clause)
                cut = np.concatenate([[0], np.cumsum(counts)])
                dests = [tid for tid, _, _, _, _ in pending]
                for d, tid in enumerate(dests):
                    if counts[d]:
                        batches.append((tid, _ReportBatch(eids[cut[d]:cut[d + 1]], masks[cut[d]:cut[d + 1]],
                                                          arena, keep)))
                n_rep = int(cut[-1])
                if self.config.trace:  # the trace keeps Report objects in emission order (engine.py:403-464)
                    dest_of = np.repeat(np.asarray(dests, np.int64), counts)
                    brank = self._rank_of_size[arena.size[eids]]
                    order = np.lexsort((groups, eids, brank, groups // self.config.group_width))
                    emitted = [Report(int(dest_of[i]), arena.lits_of(int(eids[i])), int(eids[i]), int(masks[i]))
                               for i in order.tolist()]

        if n_rep:
            with self._queue_lock:
                for d, batch in batches:
                    self._reports.setdefault(d, deque()).append(batch)
                    self._pending_reports[d] = self._pending_reports.get(d, 0) + len(batch)
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
                           for _, _, _, snaps, _ in pending for s in snaps],
                store=store_snapshot, reports=emitted))

        self.counters["rounds"] += 1
        done = time.perf_counter()
        self.counters["busy_seconds"] += done - started
        ph["rest"] = done
        t, self.last_phases = started, {}
        for k, v in ph.items():
            self.last_phases[k] = (v - t) * 1e3
            t = v
        return result

    def _round(self, gl: np.ndarray, gt: np.ndarray) -> _lib.tsg_round_result:
        """Prepare on every shard, encode on the first, copy its tables to the
        others over NVLink, launch all, collect all; the figures summed."""
        s0 = self._shards[0]
        if len(self._shards) == 1:  # one C call: prepare + encode + launch + collect
            res = s0.round(gl, gt, self._activity_inc)
            self._shard_reports = [res.reports]
            return res
        for s in self._shards:
            s.prepare(gl, gt)
        s0.encode()
        for s in self._shards[1:]:
            s.tables_from(s0)
        for s in self._shards:
            s.launch(self._activity_inc)
        rs = [s.collect() for s in self._shards]
        self._shard_reports = [r.reports for r in rs]
        res = rs[0]
        for r in rs[1:]:
            for f in ("reports", "clauses_tested", "aggregate_tests", "aggregate_tests_negative", "lane_tests",
                      "lane_triggers"):
                setattr(res, f, getattr(res, f) + getattr(r, f))
            res.reruns += r.reruns
        return res

    def _fetch_ordered(self, n: int, n_dest: int):
        """The round's records in delivery order (tsg_fetch_ordered), in a
        page-locked buffer the report batches view."""
        eid_bytes = 4 if self._next_id < (1 << 31) else 8
        mask_bytes = 4 if self.config.lane_width <= 32 else 8
        e_sec = (n * eid_bytes + 255) // 256 * 256
        buf = self._pinned.get(e_sec + n * mask_bytes)
        base = buf.p.value
        eids = np.ctypeslib.as_array(C.cast(base, C.POINTER(C.c_int32 if eid_bytes == 4 else C.c_int64)), shape=(n,))
        masks = np.ctypeslib.as_array(C.cast(base + e_sec, C.POINTER(C.c_uint32 if mask_bytes == 4 else C.c_uint64)),
                                      shape=(n,))
        groups = np.empty(n, np.int32) if self.config.trace else None
        counts = np.zeros(max(n_dest, 1), np.int64)
        got = C.c_int64(0)
        hs = (C.c_void_p * len(self._shards))(*[s.h.value for s in self._shards])
        check(self._L.tsg_fetch_ordered(hs, len(self._shards), ptr(self._rank_of_size), self._rank_of_size.size,
                                        C.c_void_p(base), eid_bytes, C.c_void_p(base + e_sec), mask_bytes,
                                        ptr(groups), ptr(counts), n, C.byref(got)))
        return eids[:got.value], masks[:got.value], groups, counts[:n_dest], buf

    def _ring_ordered(self, gt: np.ndarray, dests: List[int]):
        """The round's records from the shards' host rings (drained by their
        threads while the kernels ran), put in the delivery order
        tsg_fetch_ordered produces on the GPU: destination, chunk, bucket
        creation rank, engine id, group (engine.py:403-464)."""
        parts = [d.take(n) for d, n in zip(self._drainers, self._shard_reports) if n]
        return self._host_ordered(_reports.decode(np.concatenate(parts) if len(parts) > 1 else parts[0]), gt, dests)

    def _host_ordered(self, dec: np.ndarray, gt: np.ndarray, dests: List[int]):
        """Decoded records (reports.decode) in delivery order, on the host."""
        eid = dec["engine_id"].astype(np.int64)
        grp = dec["group"].astype(np.int32)
        dest = np.searchsorted(np.asarray(dests, np.int64), gt[grp].astype(np.int64))
        rank = self._rank_of_size[self._arena.size[eid]]
        chunk = grp // self.config.group_width
        fields = (dest, chunk, rank, eid, grp)  # most significant first
        widths = [max(int(f.max()), 0).bit_length() for f in fields]
        if sum(widths) <= 64:  # one packed key (unique per record), as the GPU ordering packs it
            key = np.zeros(len(eid), np.uint64)
            for f, w in zip(fields, widths):
                key = (key << np.uint64(w)) | f.astype(np.uint64)
            order = np.argsort(key)
        else:
            order = np.lexsort(fields[::-1])
        counts = np.bincount(dest, minlength=len(dests)).astype(np.int64)
        return eid[order], dec["lane_mask"][order], grp[order], counts, None

    def reduce_store(self) -> int:
        """engine.py:469-505; selection and compaction run on the GPU(s),
        exact across shards."""
        total = len(self.store)
        if total == 0:
            self._reduce_watermark = self._next_id
            return 0
        target = int(total * (1.0 - self.config.reduce_keep_fraction))
        if len(self._shards) == 1:
            gone = self._shards[0].reduce(self._reduce_watermark, target)
            removed = len(gone)
        else:
            removed, gone = _sharded.global_reduce(self._shards, self._reduce_watermark, target)
        self._arena.remove(gone)
        with self._id_lock:
            self._reduce_watermark = self._next_id
        self.counters["reduces"] += 1
        self.counters["clauses_removed"] += removed
        return removed

    def remove_clauses(self, engine_ids: Sequence[int]) -> int:
        """Explicit deletion (streaming config C4); order-preserving like
        _SizeBucket.compact (engine.py:184-200).  Ids still staged (added since
        the last round) or already gone are ignored."""
        ids = np.asarray(list(engine_ids), dtype=np.int64)
        if ids.size == 0:
            return 0
        removed = sum(s.remove(ids) for s in self._shards)
        self._arena.remove(ids)  # (ids not stored yet are not in the arena either)
        self.counters["clauses_deleted"] = self.counters.get("clauses_deleted", 0) + removed
        return removed

    def serve(self, stop: threading.Event, idle_sleep: float = 0.0005) -> None:
        while not stop.is_set():
            result = self.run_round()
            if result.assignments_consumed == 0:
                time.sleep(idle_sleep)

    def raw_counters(self) -> dict:
        out = dict(self.counters)
        out["store_size"] = len(self.store)
        with self._id_lock:
            out["staged_pending"] = sum(len(b.lens) if isinstance(b, _Run) else len(b[0]) for b in self._staged)
        with self._queue_lock:
            out["reports_pending"] = sum(self._pending_reports.values())
            queues = list(self._squeues.values())
        out["snapshots_pending"] = sum(q.n + len(q.bad) for q in queues)
        return out
