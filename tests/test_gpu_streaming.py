"""Streaming mode: interleaved clause adds, explicit
deletes, reduce/compaction and snapshot batches, round after round.

* `test_streaming_parity_vs_oracle_engine`: the GPU Engine and the oracle's
  restatement of the reference engine (oracle/oracle.py OracleEngine,
  engine.py:257-525) are fed the identical operation stream; every round's
  RoundResult, every thread's drained reports (in order), the counters and
  the store contents (fp64 activities bit-exact) must agree.
* `test_concurrent_producers_trace_sound_and_complete`: 32 producer threads
  submit and add while the worker serves; every traced round's reports must
  equal the oracle's reports for that round's store and snapshots
  (acceptance gate 6 of the reference, test_acceptance.py:382-442).
"""
import threading
import time

import numpy as np
import pytest

from gpu_util import require_device
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    require_device()
    import paper_2012_03119_b200 as P
    return P


def random_clause(rng, nv, lo=0, hi=14):
    s = int(rng.integers(lo, hi + 1))
    vs = rng.choice(nv, s, replace=False) + 1
    return tuple(int(v) * (1 if b else -1) for v, b in zip(vs, rng.integers(0, 2, s)))


def random_values(rng, nv):
    v = rng.choice(np.array([1, -1, 0], np.int8), size=nv + 1, p=[0.3, 0.3, 0.4])
    v[0] = 0
    return v


def store_of_engine(eng):
    return [(eid, tuple(l), o, float(a).hex()) for eid, l, o, a in eng.store.clauses()]


def store_of_oracle(ora):  # ClauseStore.clauses order (engine.py:221-231): size, then slot
    return [(eid, l, o, float(a).hex()) for eid, l, o, a in ora.store.clauses()]


@pytest.mark.parametrize("seed,lw,gw,threads,cap,max_clauses,devices", [
    (1, 8, 4, 6, 20, 3000, None),     # multi-chunk rounds, capacity reduces
    (2, 32, 32, 32, 64, 5000, None),  # the C4 shape: 32 threads, 64-deep queues -> 2 chunks
    (3, 5, 64, 9, 11, 800, None),     # tiny store: reduce inside integrate, drops
    (1, 8, 4, 6, 20, 3000, [0, 0]),   # two clause shards (exact global reduce, merged records)
    (2, 32, 32, 32, 64, 5000, [0, 0, 0]),
])
def test_streaming_parity_vs_oracle_engine(P, seed, lw, gw, threads, cap, max_clauses, devices):
    nv = 300
    cfg = dict(max_clauses=max_clauses, lane_width=lw, group_width=gw, assignment_queue_capacity=cap)
    eng = P.Engine(nv, threads, P.EngineConfig(**cfg, devices=devices))
    ora = O.OracleEngine(nv, threads, **cfg)
    rng = np.random.default_rng(seed)
    for r in range(14):
        for _ in range(int(rng.integers(20, max_clauses // 3))):
            lits = random_clause(rng, nv)
            origin = int(rng.integers(0, threads))
            assert eng.add_clause(lits, origin) == ora.add_clause(lits, origin)
        if r % 3 == 2:  # explicit deletes, including ids that are staged or long gone
            ids = rng.integers(0, max(1, ora.next_id), 200)
            assert eng.remove_clauses(ids) == ora.remove_clauses(ids)
        for t in range(threads):
            for _ in range(int(rng.integers(0, cap + 4))):
                v = random_values(rng, nv)
                seq = int(rng.integers(0, 1 << 30))
                assert eng.submit_assignment(P.AssignmentSnapshot(t, v, seq)) == ora.submit_assignment(t, v, seq)
        if r % 4 == 3:
            assert eng.reduce_store() == ora.reduce_store()
        res = eng.run_round()
        ores = ora.run_round()
        assert [res.reports_emitted, res.clauses_tested, res.assignments_consumed,
                res.aggregate_tests_negative] == [ores["reports_emitted"], ores["clauses_tested"],
                                                  ores["assignments_consumed"],
                                                  ores["aggregate_tests_negative"]], r
        for t in range(threads):
            got = [(r_.destination, r_.lits, r_.engine_id, r_.lane_mask) for r_ in eng.drain_reports(t)]
            want = [(o.destination, o.lits, o.engine_id, o.lane_mask) for o in ora.drain_reports(t)]
            assert got == want, (r, t)
        c = eng.raw_counters()
        for k, v in ora.counters.items():
            assert c[k] == v, (r, k)
        assert store_of_engine(eng) == store_of_oracle(ora), r
    eng.close()


def test_wrong_length_snapshot_raises_at_round(P):
    # the reference accepts any snapshot and fails when the round packs it
    # (bitpack.py:99-103)
    eng = P.Engine(10, 2)
    eng.add_clause((1, 2), origin=0)
    assert eng.submit_assignment(P.AssignmentSnapshot(0, np.zeros(5, np.int8), 0))
    with pytest.raises(ValueError):
        eng.run_round()
    eng.close()


def test_concurrent_producers_trace_sound_and_complete(P):
    nv, threads = 2000, 32
    eng = P.Engine(nv, threads, P.EngineConfig(trace=True, max_clauses=20_000, assignment_queue_capacity=64))
    stop = threading.Event()
    worker = threading.Thread(target=eng.serve, args=(stop,))
    worker.start()

    def producer(t):
        rng = np.random.default_rng(1000 + t)
        for i in range(120):
            if rng.random() < 0.5:
                eng.add_clause(random_clause(rng, nv, 1, 8), origin=t)
            eng.submit_assignment(P.AssignmentSnapshot(t, random_values(rng, nv), i))
            if i % 10 == 0:
                eng.drain_reports(t)
                time.sleep(0.001)

    ps = [threading.Thread(target=producer, args=(t,)) for t in range(threads)]
    for p in ps:
        p.start()
    for p in ps:
        p.join()
    time.sleep(0.2)
    stop.set()
    worker.join(timeout=60)
    assert not worker.is_alive()
    c = eng.raw_counters()
    assert c["snapshots_pending"] == 0 and c["snapshots_consumed"] == c["snapshots_accepted"]
    checked = 0
    for tr in eng.trace:
        if not tr.snapshots:
            continue
        # regroup like engine.py:390-399: tids ascending, submission order within a tid
        by_tid = {}
        for tid, values in tr.snapshots:
            by_tid.setdefault(tid, []).append(values)
        rows, lanes, tids = [], [], []
        for tid in sorted(by_tid):
            s = by_tid[tid]
            for i in range(0, len(s), 32):
                rows.extend(s[i:i + 32])
                lanes.append(len(s[i:i + 32]))
                tids.append(tid)
        st = O.OracleStore()
        for eid, lits in tr.store:
            st.insert(list(lits), eid, 0, 1.0)
        recs, _ = st.test_round(nv, np.stack(rows), lanes, tids, 32, 32, 1.0)
        want = sorted((tids[int(r["group"])], int(r["engine_id"]), int(r["lane_mask"])) for r in recs)
        got = sorted((r.destination, r.engine_id, r.lane_mask) for r in tr.reports)
        assert got == want
        checked += 1
    assert checked > 0
    eng.close()
