"""Pure host logic of the product, on CPU: the strong-scaling shard split
(workload.shard) and the Engine's append-only literal arena (Report.lits
stay valid for a batch after later inserts grow the arena)."""
import numpy as np


def test_shard_split_is_a_partition_with_global_ids():
    from paper_2012_03119_b200 import workload as W
    b = W.clause_buckets(5000, 300, np.random.default_rng(1), 1, 9)
    flat, offs, ids = W.flatten(b)
    want = {int(i): tuple(flat[offs[k]:offs[k + 1]].tolist()) for k, i in enumerate(ids)}
    for world in (1, 2, 3, 8):
        got = {}
        for r in range(world):
            f, o, i = W.shard(b, world, r)
            assert np.all(np.diff(i) > 0)  # engine ids ascend within a shard (tsg_add_clauses)
            for k, e in enumerate(i.tolist()):
                assert e not in got
                got[e] = tuple(f[o[k]:o[k + 1]].tolist())
            # every size bucket balanced across the ranks
            sizes = np.diff(o)
            for s, arr in b.items():
                share = int((sizes == s).sum())
                assert abs(share - arr.shape[0] / world) <= 1
        assert got == want


def test_arena_keeps_round_literals():
    from paper_2012_03119_b200.engine import _Arena
    a = _Arena()
    rng = np.random.default_rng(2)
    ref = {}
    snaps = []
    nxt = 0
    for r in range(30):
        n = int(rng.integers(1, 400))
        lens = rng.integers(0, 12, n).astype(np.int32)
        flat = rng.integers(-50, 50, int(lens.sum())).astype(np.int32)
        ids = np.arange(nxt, nxt + n, dtype=np.int64)
        nxt += n
        a.append(ids, lens, flat)
        o = 0
        for i, s in zip(ids.tolist(), lens.tolist()):
            ref[i] = tuple(flat[o:o + s].tolist())
            o += s
        snaps.append((a.snapshot(), nxt))
    for snap, upto in snaps:  # every round's arena still answers for the ids it knew
        for i in rng.integers(0, upto, 50).tolist():
            assert snap.lits_of(i) == ref[i]


def test_literal_arena_reclaims_removed_clauses_without_touching_old_batches():
    # engine.py's Report-literal arena: appends, removals, compaction; a view
    # taken for a round's report batch keeps its literals through all of it
    import numpy as np
    from paper_2012_03119_b200.engine import _Arena
    rng = np.random.default_rng(3)

    class Small(_Arena):  # reclaim at any size, and count the rebuilds
        RECLAIM_MIN = 0
        rebuilds = 0

        def _compact(self):
            Small.rebuilds += 1
            super()._compact()

    a = Small()
    want = {}
    nxt = 0
    views = []
    for rnd in range(30):
        n = int(rng.integers(1, 4000))
        lens = rng.integers(2, 31, n).astype(np.int32)
        flat = rng.integers(-500, 500, int(lens.sum())).astype(np.int32)
        ids = np.arange(nxt, nxt + n, dtype=np.int64)
        nxt += n
        a.append(ids, lens, flat)
        o = 0
        for i, L in zip(ids.tolist(), lens.tolist()):
            want[i] = tuple(flat[o:o + L].tolist())
            o += L
        view = a.snapshot()
        sample = rng.choice(nxt, min(50, nxt), replace=False)
        views.append((view, {int(i): want[int(i)] for i in sample if int(i) in want}))
        gone = rng.choice(nxt, nxt // 3, replace=False)
        a.remove(gone)
        a.remove(gone[:10])  # twice: ignored
        for i in gone.tolist():
            want.pop(i, None)
    assert Small.rebuilds > 3 and a.dead_lits <= a.live_lits  # reclaimed along the way
    assert a.used <= 2 * a.live_lits
    for i, lits in want.items():
        assert a.lits_of(i) == lits
    for view, expect in views:  # old batches: literals as of their round
        for i, lits in expect.items():
            assert view.lits_of(i) == lits


def test_ring_drainer_reassembles_runs_in_ring_order():
    # native.RingDrainer: several threads drain runs of ring positions in any
    # order; take(n) must return exactly the next n positions -- one
    # round's records, then the next's
    import threading
    import numpy as np
    from paper_2012_03119_b200._lib import REPORT_DTYPE
    from paper_2012_03119_b200.native import RingDrainer

    total = 5000
    rng = np.random.default_rng(5)
    cuts = np.unique(np.concatenate([[0, total], rng.integers(1, total, 300)]))
    runs = [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:])]
    order = rng.permutation(len(runs))  # handed out in random order to random threads

    class FakeEngine:
        def __init__(self):
            self.lock = threading.Lock()
            self.i = 0

        def ring_drain(self, max_records, timeout_ms=0.0, out=None, with_pos=False):
            with self.lock:
                if self.i >= len(order):
                    time.sleep(0.001)
                    return np.zeros(0, REPORT_DTYPE), -1
                a, b = runs[order[self.i]]
                self.i += 1
            recs = np.zeros(b - a, REPORT_DTYPE)
            recs["key"] = np.arange(a, b, dtype=np.uint64)  # the record's position, as its payload
            time.sleep(float(rng.random()) * 1e-4)
            return recs, a

    import time
    dr = RingDrainer(FakeEngine(), threads=4, batch=64)
    try:
        got, pos = [], 0
        for n in (1, 777, 0, 1500, 2222, total - 4500):  # "rounds" of these sizes
            part = dr.take(n, timeout_s=10)
            assert len(part) == n
            assert np.array_equal(part["key"], np.arange(pos, pos + n, dtype=np.uint64))
            pos += n
    finally:
        dr.close()


def test_engine_host_ordering_matches_the_reference_order():
    # Engine._host_ordered (report ring path): records into delivery order --
    # destination, chunk, bucket creation rank, engine id, group
    # (engine.py:403-464) -- from one packed 64-bit key
    import numpy as np
    from paper_2012_03119_b200 import reports
    from paper_2012_03119_b200.engine import Engine, EngineConfig, _Arena
    rng = np.random.default_rng(9)
    for n_ids, n_groups, gw in ((5000, 40, 8), (2_000_000, 3000, 64)):
        e = object.__new__(Engine)
        e.config = EngineConfig(group_width=gw)
        n = 3000
        eids = rng.choice(n_ids, n, replace=False).astype(np.int64)
        sizes = rng.integers(1, 30, n).astype(np.int32)
        e._arena = _Arena()
        e._arena.size = np.zeros(n_ids, np.int32)
        e._arena.size[eids] = sizes  # only the size lookups matter here
        e._rank_of_size = rng.permutation(64).astype(np.int32)
        gt = np.sort(rng.integers(0, 7, n_groups)).astype(np.int32)  # a thread's groups are consecutive
        dec = np.zeros(n, reports.DECODED_DTYPE)
        dec["engine_id"] = eids
        dec["group"] = rng.integers(0, n_groups, n)
        dec["lane_mask"] = rng.integers(1, 1 << 32, n, dtype=np.uint64)
        dests = sorted(set(gt.tolist()))
        got_e, got_m, got_g, counts, _ = e._host_ordered(dec, gt, dests)
        dest = np.searchsorted(np.asarray(dests), gt[dec["group"]])
        want = np.lexsort((dec["group"], dec["engine_id"], e._rank_of_size[sizes], dec["group"] // gw, dest))
        assert np.array_equal(got_e, dec["engine_id"][want])
        assert np.array_equal(got_g, dec["group"][want])
        assert np.array_equal(got_m, dec["lane_mask"][want])
        assert np.array_equal(counts, np.bincount(dest, minlength=len(dests)))
