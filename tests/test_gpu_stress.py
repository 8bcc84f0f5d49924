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
