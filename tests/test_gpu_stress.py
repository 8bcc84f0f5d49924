"""Randomised parity of the GPU engine against the CPU oracle: random store
sizes, clause sizes (empty and long clauses included), lane / group widths,
thread counts, activity increments, egress formats and several rounds per
store; records (engine id, lane mask, group) in the reference order,
counters and the final store with fp64 activities must be identical.

TSG_STRESS_SECONDS (default 20) sets the run time; TSG_STRESS_SEED the seed.
profiles/r01_stress_async.md records a 7-minute run.
"""
import os
import time

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_randomised_parity_vs_oracle():
    from gpu_util import require_device
    require_device()
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    secs = float(os.environ.get("TSG_STRESS_SECONDS", "20"))
    seed = int(os.environ.get("TSG_STRESS_SEED", "7"))
    rng = np.random.default_rng(seed)
    t_end = time.time() + secs
    cases = rounds_done = 0
    while time.time() < t_end:
        lw = int(rng.choice([32, 32, 16, 64, 7, 1]))
        gw = int(rng.choice([32, 32, 8, 64, 3]))
        nv = int(rng.choice([50, 300, 5000, 40000]))
        n = int(rng.integers(100, 60000))
        lo, hi = (0, 12) if rng.random() < 0.5 else (2, 30)
        if rng.random() < 0.1 and nv >= 300:
            lo, hi = 60, 120
        hi = min(hi, nv)
        threads = int(rng.integers(1, 9))
        lanes = int(rng.integers(1, 80))
        buckets = W.clause_buckets(n, nv, rng, lo, hi)
        flat, offs, ids = W.flatten(buckets)
        org = (ids % 5).astype(np.int32)
        dev = NativeEngine(nv, lw, gw)
        if lw <= 32 and rng.random() < 0.5:
            dev.set_record_bytes(12)
        all_pairs = rng.random() < 0.3  # every triggering (clause, group): the oracle with a thread per group
        dev.set_all_pairs(all_pairs)
        dev.add_clauses(flat, offs, ids, org, 1.0)
        ora = O.OracleStore()
        k = 0
        for s, arr in buckets.items():
            for row in arr:
                ora.insert(row.tolist(), int(ids[k]), int(org[k]), 1.0)
                k += 1
        inc = float(rng.uniform(0.5, 3.0))
        for r in range(int(rng.integers(1, 4))):
            snaps = W.snapshots(threads, lanes, nv, rng)
            gl, gt = W.groups_for(threads, lanes, lw)
            dev.stage(snaps)
            try:
                res = dev.round(gl, gt, inc)
            except Exception as exc:
                raise AssertionError(f"case {cases} round {r}: lw {lw} gw {gw} nv {nv} n {n} sizes {lo}-{hi} "
                                     f"threads {threads} lanes {lanes} store {len(dev)}: {exc}") from exc
            recs = dev.fetch(res.reports)
            ogt = np.arange(len(gl), dtype=np.int32) if all_pairs else gt
            orecs, octr = ora.test_round(nv, snaps, gl, ogt, lw, gw, inc, nthreads=8)
            recs = W.in_reference_order(recs, offs, ids, buckets, gw)
            assert len(recs) == len(orecs), (len(recs), len(orecs), lw, gw, nv, n)
            for f in ("engine_id", "lane_mask", "group"):
                assert np.array_equal(recs[f], orecs[f]), f
            for f in ("clauses_tested", "aggregate_tests", "aggregate_tests_negative", "lane_tests", "lane_triggers"):
                assert getattr(res, f) == octr[f], f
            inc /= 0.999
            rounds_done += 1
        for (s, lits, ids_d, org_d, acts_d), (s2, n2, lits2, ids2, org2, acts2) in zip(dev.buckets(), ora.buckets()):
            assert s == s2 and np.array_equal(lits, lits2) and np.array_equal(ids_d, ids2)
            assert np.array_equal(acts_d.view(np.uint64), acts2.view(np.uint64))
        dev.close()
        cases += 1
    print(f"parity ok: {cases} stores, {rounds_done} rounds, seed {seed}")
    assert cases > 0


def test_randomised_engine_streams_vs_oracle_engine():
    """The drop-in Engine under random operation streams (adds, explicit
    deletes, reduces, snapshot bursts that overflow queues, wrong-free
    rounds) against the oracle's restatement of the reference engine, with
    random word widths, 1-3 clause shards, the chunk filter on or off and
    the records through the device buffer or the host report ring:
    every round's result, every thread's drained reports in order, the
    counters and the store (fp64 activities bit-exact)."""
    from gpu_util import require_device
    require_device()
    import paper_2012_03119_b200 as P
    secs = float(os.environ.get("TSG_STRESS_SECONDS", "20"))
    seed = int(os.environ.get("TSG_STRESS_SEED", "7"))
    rng = np.random.default_rng(seed + 1)
    t_end = time.time() + secs
    streams = rounds_done = 0
    while time.time() < t_end:
        nv = int(rng.choice([20, 200, 3000]))
        threads = int(rng.integers(1, 7))
        lw = int(rng.choice([1, 4, 16, 32, 64]))
        gw = int(rng.choice([1, 3, 8, 32, 64]))
        cap = int(rng.integers(1, 3 * lw + 2))
        max_clauses = int(rng.integers(50, 4000))
        devices = [None, [0, 0], [0, 0, 0]][int(rng.integers(0, 3))]
        chunk_filter = bool(rng.random() < 0.5)
        ring = int(rng.choice([0, 0, 256, 4096])) if lw <= 32 else 0  # records through the host report ring
        cfg = dict(max_clauses=max_clauses, lane_width=lw, group_width=gw, assignment_queue_capacity=cap)
        eng = P.Engine(nv, threads, P.EngineConfig(**cfg, devices=devices, chunk_filter=chunk_filter,
                                                   report_ring=ring))
        ora = O.OracleEngine(nv, threads, **cfg)
        hi = min(nv, 14)
        for r in range(int(rng.integers(2, 8))):
            for _ in range(int(rng.integers(0, max_clauses // 2 + 2))):
                s = int(rng.integers(0, hi + 1))
                vs = rng.choice(nv, s, replace=False) + 1
                lits = tuple(int(v) * (1 if b else -1) for v, b in zip(vs, rng.integers(0, 2, s)))
                o = int(rng.integers(0, threads))
                assert eng.add_clause(lits, o) == ora.add_clause(lits, o)
            if rng.random() < 0.3:
                ids = rng.integers(0, max(1, ora.next_id), int(rng.integers(1, 200)))
                assert eng.remove_clauses(ids) == ora.remove_clauses(ids)
            for t in range(threads):
                for _ in range(int(rng.integers(0, cap + 3))):
                    v = rng.choice(np.array([1, -1, 0], np.int8), size=nv + 1, p=[0.3, 0.3, 0.4])
                    v[0] = 0
                    assert eng.submit_assignment(P.AssignmentSnapshot(t, v, 0)) == ora.submit_assignment(t, v, 0)
            if rng.random() < 0.2:
                assert eng.reduce_store() == ora.reduce_store()
            res, ores = eng.run_round(), ora.run_round()
            ctx = (streams, r, nv, threads, lw, gw, cap, max_clauses, devices, chunk_filter, ring)
            assert [res.reports_emitted, res.clauses_tested, res.assignments_consumed,
                    res.aggregate_tests_negative] == [ores["reports_emitted"], ores["clauses_tested"],
                                                      ores["assignments_consumed"],
                                                      ores["aggregate_tests_negative"]], ctx
            for t in range(threads):
                got = [(x.destination, x.lits, x.engine_id, x.lane_mask) for x in eng.drain_reports(t)]
                want = [(x.destination, x.lits, x.engine_id, x.lane_mask) for x in ora.drain_reports(t)]
                assert got == want, ctx
            c = eng.raw_counters()
            for k, v in ora.counters.items():
                assert c[k] == v, (ctx, k)
            rounds_done += 1
        got = [(eid, tuple(l), o, float(a).hex()) for eid, l, o, a in eng.store.clauses()]
        want = [(eid, l, o, float(a).hex()) for eid, l, o, a in ora.store.clauses()]
        assert got == want, (streams, nv, threads, lw, gw, devices)
        eng.close()
        streams += 1
    print(f"engine streams ok: {streams} streams, {rounds_done} rounds, seed {seed}")
    assert streams > 0
