"""Host report ring (north_star subsystem 4, include/tsg.h tsg_ring_*): the
trigger kernel writes records straight into page-locked host memory and CPU
threads drain them while it runs.

Parity bar: the drained records of a round, put in the reference's emission
order, are bit-identical to the CPU oracle's (engine.py:437-467 semantics,
all-pairs = multi_trigger's pair set), and to the device-buffer path of the
same round; counters are unchanged.  A ring smaller than one flush's worth
of records wraps many times per round; a ring nobody drains fails the round
within its wait bound instead of hanging."""
import os
import time

import numpy as np
import pytest

from gpu_util import require_device
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    require_device()
    from paper_2012_03119_b200 import workload as W
    return W


def store(W, n, nv, seed, lw=32, gw=32):
    from paper_2012_03119_b200.native import NativeEngine
    rng = np.random.default_rng(seed)
    buckets = W.clause_buckets(n, nv, rng)
    flat, offs, ids = W.flatten(buckets)
    eng = NativeEngine(nv, lw, gw, report_capacity=1 << 16)
    eng.add_clauses(flat, offs, ids)
    return eng, rng, buckets, flat, offs, ids


def decoded(raw):
    from paper_2012_03119_b200 import reports
    return reports.decode(raw)


def as_set(dec):
    return set(zip(dec["engine_id"].tolist(), dec["group"].tolist(), dec["lane_mask"].tolist()))


@pytest.mark.parametrize("all_pairs", [False, True])
@pytest.mark.parametrize("drainers", [1, 3])
def test_ring_parity_vs_oracle(W, all_pairs, drainers):
    from paper_2012_03119_b200.native import RingDrainer
    c = W.CONFIGS["C1"]
    eng, rng, buckets, flat, offs, ids = store(W, c.n_clauses, c.num_vars, c.seed)
    if all_pairs:
        eng.set_all_pairs(True)
    ora = O.OracleStore()
    ora.insert_flat(flat, offs, ids)
    eng.ring_open(capacity=4096)
    dr = RingDrainer(eng, threads=drainers, batch=512)
    try:
        for r in range(2):
            snaps = W.snapshots(c.threads, c.lanes, c.num_vars, rng)
            gl, gt = W.groups_for(c.threads, c.lanes, 32)
            eng.stage(snaps)
            res = eng.round(gl, gt, 1.0)
            got = W.in_reference_order(decoded(dr.take(res.reports)), offs, ids, buckets, 32)
            ogt = np.arange(len(gl), dtype=np.int32) if all_pairs else gt
            orecs, octr = ora.test_round(c.num_vars, snaps, gl, ogt, 32, 32, 1.0, nthreads=os.cpu_count() or 8)
            assert res.reports == len(orecs) > 0
            for f in ("engine_id", "lane_mask", "group"):
                assert np.array_equal(got[f], orecs[f]), f
            assert res.lane_triggers == octr["lane_triggers"]
            assert res.aggregate_tests_negative == octr["aggregate_tests_negative"]
        exp, con, failed = eng.ring_status()
        assert exp == con and not failed
    finally:
        dr.close()
        eng.ring_close()
        eng.close()


def test_ring_wraps_and_matches_device_buffer(W):
    """A 128-record ring (one flush) under a round of tens of thousands of
    records: the kernel's warps wait for the drainer lap after lap."""
    from paper_2012_03119_b200 import _lib
    from paper_2012_03119_b200.native import RingDrainer
    eng, rng, buckets, flat, offs, ids = store(W, 200_000, 20_000, 5)
    eng.set_all_pairs(True)
    snaps = W.snapshots(4, 32, 20_000, rng)
    gl, gt = W.groups_for(4, 32, 32)
    eng.stage(snaps)
    ref = eng.round(gl, gt, 1.0)
    want = as_set(eng.fetch(ref.reports))
    assert ref.reports > 10_000  # > 80 laps of the ring
    eng.ring_open(capacity=128, wait_ms=10_000)
    dr = RingDrainer(eng, threads=2, batch=64)
    try:
        res = eng.round(gl, gt, 1.0)
        got = decoded(dr.take(res.reports))
        assert res.reports == ref.reports and res.lane_triggers == ref.lane_triggers
        assert len(as_set(got)) == len(got) and as_set(got) == want
        with pytest.raises(ValueError, match="ring"):  # ringed rounds have no device records
            eng.fetch_raw(1)
    finally:
        dr.close()
        eng.ring_close()
    # closed: the device buffer path again
    res = eng.round(gl, gt, 1.0)
    assert as_set(eng.fetch(res.reports)) == want
    eng.close()


@pytest.mark.parametrize("drainers,cap", [(1, 1 << 12), (4, 1 << 12), (3, 256)])
def test_ring_two_rounds_in_flight(W, drainers, cap):
    """launch A, launch B, collect both: the ring positions of A's records
    all precede B's (B's kernel reserves after A's finished), and take()
    reassembles the drainer threads' runs in position order -- A's records,
    then B's, however many threads drain."""
    from paper_2012_03119_b200.native import RingDrainer, pack_rows
    nv = 5000
    eng, rng, buckets, flat, offs, ids = store(W, 60_000, nv, 9)
    rounds = []
    for _ in range(2):
        snaps = W.snapshots(3, 32, nv, rng)
        gl, gt = W.groups_for(3, 32, 32)
        eng.stage(snaps)
        res = eng.round(gl, gt, 1.0)
        rounds.append((pack_rows(snaps, nv), gl, gt, as_set(eng.fetch(res.reports)), res.reports))
    eng.ring_open(capacity=cap)
    dr = RingDrainer(eng, threads=drainers, batch=256)
    try:
        for packed, gl, gt, _, _ in rounds:
            eng.stage_packed(packed)
            eng.prepare(gl, gt)
            eng.encode()
            eng.launch(1.0)
        counts = [eng.collect().reports for _ in rounds]
        assert counts == [r[4] for r in rounds]
        for (_, _, _, want, n), k in zip(rounds, counts):
            assert as_set(decoded(dr.take(k))) == want
    finally:
        dr.close()
        eng.ring_close()
        eng.close()


def test_undrained_ring_fails_within_its_wait_bound(W):
    from paper_2012_03119_b200 import _lib
    from paper_2012_03119_b200.native import RingDrainer
    eng, rng, buckets, flat, offs, ids = store(W, 200_000, 20_000, 5)
    eng.set_all_pairs(True)
    snaps = W.snapshots(4, 32, 20_000, rng)
    gl, gt = W.groups_for(4, 32, 32)
    eng.stage(snaps)
    eng.ring_open(capacity=128, wait_ms=50)
    t0 = time.monotonic()
    with pytest.raises(_lib.CapacityError, match="dropped"):
        eng.round(gl, gt, 1.0)
    assert time.monotonic() - t0 < 30
    assert eng.ring_status()[2]  # failed, and stays failed
    with pytest.raises(_lib.CapacityError):
        eng.round(gl, gt, 1.0)
    eng.ring_close()
    eng.ring_open(capacity=1 << 16)  # reopened: a fresh ring works
    dr = RingDrainer(eng)
    try:
        res = eng.round(gl, gt, 1.0)
        assert len(dr.take(res.reports)) == res.reports > 0
    finally:
        dr.close()
        eng.ring_close()
        eng.close()


def test_ring_argument_checks(W):
    from paper_2012_03119_b200.native import NativeEngine
    e64 = NativeEngine(100, 64, 32)
    with pytest.raises(ValueError, match="lane_width"):
        e64.ring_open(1024)
    e64.close()
    e = NativeEngine(100, 32, 32)
    with pytest.raises(ValueError):
        e.ring_drain(1)  # no ring open
    with pytest.raises(ValueError):
        e.ring_open(16)  # below one flush
    e.ring_open(1000)
    with pytest.raises(ValueError):
        e.ring_open(1000)  # already open
    assert len(e.ring_drain(8, timeout_ms=1)) == 0
    e.ring_close()
    e.close()


def test_ring_close_while_drainers_run(W):
    """tsg_ring_close waits for drainers inside tsg_ring_drain; later drain
    calls fail cleanly (no use of the freed ring)."""
    from paper_2012_03119_b200.native import RingDrainer
    eng, rng, buckets, flat, offs, ids = store(W, 50_000, 3000, 3)
    snaps = W.snapshots(3, 32, 3000, rng)
    gl, gt = W.groups_for(3, 32, 32)
    eng.stage(snaps)
    eng.ring_open(capacity=1 << 12)
    dr = RingDrainer(eng, threads=3, batch=128)
    res = eng.round(gl, gt, 1.0)
    assert len(dr.take(res.reports)) == res.reports
    eng.ring_close()  # drainers still polling
    time.sleep(0.05)
    dr.close()
    assert dr.error is None or isinstance(dr.error, ValueError)
    res = eng.round(gl, gt, 1.0)  # the device buffer path again
    assert len(eng.fetch(res.reports)) == res.reports
    eng.close()
