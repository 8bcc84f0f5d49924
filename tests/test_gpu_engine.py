"""The GPU Engine vs the reference (golden scenarios recorded from the
reference Engine itself) and vs the CPU oracle at config sizes.

Parity bar: bit-exact -- identical ordered report lists per thread,
identical counters, identical store contents with activities compared as
float.hex (engine.py:460 rounding, no FMA)."""
import threading
import time

import numpy as np
import pytest

from golden_io import engine_golden
from gpu_util import require_device
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    require_device()
    import paper_2012_03119_b200 as P
    return P


def replay(P, spec, devices=None, report_ring=0):
    eng = P.Engine(spec["num_vars"], spec["threads"], P.EngineConfig(**spec["config"], devices=devices,
                                                                     report_ring=report_ring))
    for op, exp in zip(spec["ops"], spec["expect"]):
        if op[0] == "add":
            assert eng.add_clause(op[1], origin=op[2]) == exp["id"]
        elif op[0] == "submit":
            snap = P.AssignmentSnapshot(op[1], np.asarray(op[3], dtype=np.int8), op[2])
            assert eng.submit_assignment(snap) == exp["ok"]
        else:
            if op[0] == "round":
                r = eng.run_round()
                got = [r.reports_emitted, r.clauses_tested, r.assignments_consumed, r.aggregate_tests_negative]
                assert got == exp["result"], spec["name"]
            else:
                assert eng.reduce_store() == exp["removed"], spec["name"]
            for t in spec["observe_threads"]:
                got = [[list(r.lits), r.engine_id, r.lane_mask, r.destination] for r in eng.drain_reports(t)]
                assert got == exp["reports"][str(t)], (spec["name"], t)
            counters = {k: v for k, v in eng.raw_counters().items() if k != "busy_seconds"}
            assert counters == exp["counters"], spec["name"]
            store = [[eid, list(l), o, float(a).hex()] for eid, l, o, a in eng.store.clauses()]
            assert store == exp["store"], spec["name"]
            assert [[s, b.count] for s, b in eng.store.buckets.items()] == exp["bucket_order"]
            assert float(eng._activity_inc).hex() == exp["activity_inc"]
    eng.close()


# devices [0, 0]: the store sharded over two engines (one per listed GPU;
# both on the test box's one GPU), tables copied peer to peer, records
# ordered together, reduce exact across the shards
@pytest.mark.parametrize("devices", [None, [0, 0]])
def test_reference_scenarios_bit_exact(P, devices):
    for spec in engine_golden():
        replay(P, spec, devices)


# the records through the host report ring (drainer threads, host ordering)
# instead of the device buffer: the same reference results (the ring carries
# 32-bit lane masks, so the width-64 scenarios are not eligible)
@pytest.mark.parametrize("devices", [None, [0, 0]])
def test_reference_scenarios_through_the_report_ring(P, devices):
    n = 0
    for spec in engine_golden():
        if spec["config"].get("lane_width", 32) > 32:
            continue
        replay(P, spec, devices, report_ring=256)
        n += 1
    assert n >= 10


# ---- ported from the reference's tests/test_engine.py ---------------------

def snap(P, tid, seq, nv, mapping):
    v = np.zeros(nv + 1, dtype=np.int8)
    for k, w in mapping.items():
        v[k] = w
    return P.AssignmentSnapshot(tid, v, seq)


def test_trigger_bumps_activity(P):
    e = P.Engine(2, 1)
    e.add_clause((1,), origin=0)
    e.run_round()
    bucket = e.store.buckets[1]
    before = float(bucket.activities[0])
    e.submit_assignment(snap(P, 0, 0, 2, {1: -1}))
    e.run_round()
    assert float(bucket.activities[0]) > before


def test_trace_records_snapshots_store_and_reports(P):
    e = P.Engine(2, 1, P.EngineConfig(trace=True))
    e.add_clause((1, 2), origin=0)
    e.submit_assignment(snap(P, 0, 0, 2, {1: -1, 2: -1}))
    e.run_round()
    assert len(e.trace) == 1
    t = e.trace[0]
    assert t.store == [(0, (1, 2))]
    tid, values = t.snapshots[0]
    assert tid == 0 and values[1] == -1
    assert len(t.reports) == 1


def test_serve_loop_runs_until_stopped(P):
    e = P.Engine(2, 1)
    e.add_clause((1, 2), origin=0)
    stop = threading.Event()
    w = threading.Thread(target=e.serve, args=(stop,))
    w.start()
    e.submit_assignment(snap(P, 0, 0, 2, {1: -1, 2: -1}))
    deadline = time.time() + 10
    reps = []
    while time.time() < deadline and not reps:
        reps = e.drain_reports(0)
        time.sleep(0.005)
    stop.set()
    w.join(timeout=10)
    assert not w.is_alive() and len(reps) == 1


def test_raw_counters_and_empty_round(P):
    e = P.Engine(2, 1)
    e.add_clause((1,), origin=0)
    e.submit_assignment(snap(P, 0, 0, 2, {}))
    c = e.raw_counters()
    assert c["staged_pending"] == 1 and c["snapshots_pending"] == 1 and c["reports_pending"] == 0
    e2 = P.Engine(2, 1)
    r = e2.run_round()
    assert r.assignments_consumed == 0 and r.reports_emitted == 0 and e2.counters["rounds"] == 1


def test_literal_out_of_range_raises(P):
    # the reference stores any literal and only fails when a round tests it
    # (numpy IndexError in the gather, engine.py:251)
    e = P.Engine(3, 1)
    e.add_clause((1, 7), origin=0)
    e.run_round()
    assert len(e.store) == 1
    e.submit_assignment(snap(P, 0, 0, 3, {1: -1}))
    with pytest.raises(IndexError):
        e.run_round()


# ---- config-scale parity vs the CPU oracle ---------------------------------

def run_both(P, cfg_name=None, n=None, threads=None, lanes=None, nv=None, lane_width=32, group_width=32,
             seed=0, inc=1.0, rounds=1, size_lo=2, size_hi=30, all_pairs=False, packed=False, chunk_filter=False):
    """The device engine and the oracle on the same store and snapshots.
    all_pairs: the device emits every triggering (clause, group) -- compared
    with the oracle run with one thread per group, whose one-report-per-
    (clause, thread) set is then exactly multi_trigger's pair set
    (bitpack.py:282-300; tests/test_oracle_golden.py pins the oracle to it)."""
    import os
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    if cfg_name:
        c = W.CONFIGS[cfg_name]
        n, threads, lanes, nv, seed = c.n_clauses, c.threads, c.lanes, c.num_vars, c.seed
    rng = np.random.default_rng(seed)
    buckets = W.clause_buckets(n, nv, rng, size_lo, size_hi)
    flat, offs, ids = W.flatten(buckets)
    org = (ids % 7).astype(np.int32)
    dev = NativeEngine(nv, lane_width, group_width, report_capacity=1 << 20, chunk_filter=chunk_filter)
    if all_pairs:
        dev.set_all_pairs(True)
    dev.add_clauses(flat, offs, ids, org, 1.0)
    ora = O.OracleStore()
    ora.insert_flat(flat, offs, ids, org)
    del flat
    for r in range(rounds):
        snaps = W.snapshots(threads, lanes, nv, rng)
        gl, gt = W.groups_for(threads, lanes, lane_width)
        if packed:
            from paper_2012_03119_b200.native import pack_rows
            dev.stage_packed(pack_rows(snaps, nv, threads=os.cpu_count() or 1))
        else:
            dev.stage(snaps)
        res = dev.round(gl, gt, inc)
        recs = dev.fetch(res.reports)
        ogt = np.arange(len(gl), dtype=np.int32) if all_pairs else gt
        orecs, octr = ora.test_round(nv, snaps, gl, ogt, lane_width, group_width, inc,
                                     nthreads=os.cpu_count() or 8)
        if all_pairs:
            assert len(set(gt.tolist())) < len(gl)  # threads with several groups: pairs != reports
        recs = W.in_reference_order(recs, offs, ids, buckets, group_width)
        assert len(recs) == len(orecs)
        for f in ("engine_id", "lane_mask", "group"):
            assert np.array_equal(recs[f], orecs[f]), f
        assert res.clauses_tested == octr["clauses_tested"]
        assert res.aggregate_tests == octr["aggregate_tests"]
        assert res.aggregate_tests_negative == octr["aggregate_tests_negative"]
        assert res.lane_tests == octr["lane_tests"]
        assert res.lane_triggers == octr["lane_triggers"]
        inc = inc / 0.999
    for (s, lits, ids_d, org_d, acts_d), (s2, n2, lits2, ids2, org2, acts2) in zip(dev.buckets(), ora.buckets()):
        assert s == s2 and np.array_equal(lits, lits2) and np.array_equal(ids_d, ids2)
        assert np.array_equal(org_d, org2)
        assert np.array_equal(acts_d.view(np.uint64), acts2.view(np.uint64))  # bit-exact fp64
    return res


def test_c1_parity_vs_oracle(P):
    res = run_both(P, "C1", rounds=2)
    assert res.reports > 0 and res.lane_triggers > 0


def test_c2_full_size_parity(P):
    # C2 at its full size: 1M clauses x 256 assignments (8 threads x 32), 50k vars
    res = run_both(P, "C2", packed=True)
    assert res.reports > 100_000


# pair-set parity: every triggering (clause, group) at
# the configs' full clause counts, with lane width 16 so every thread owns
# two groups (the pair set then differs from the first-per-thread reports);
# C3 at lane width 16 is 64 groups = two chunks, i.e. the chunk-level
# aggregate path at full size
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_pair_set_parity_full_size(P, cfg):
    res = run_both(P, cfg, lane_width=16, all_pairs=True, packed=True, chunk_filter=cfg == "C3")
    assert res.reports > 0 and res.n_chunks == (2 if cfg == "C3" else 1)


@pytest.mark.parametrize("lw,gw,threads,lanes", [(32, 32, 3, 40), (64, 64, 2, 64), (64, 8, 5, 70),
                                                 (7, 3, 4, 20), (1, 64, 3, 30), (32, 16, 40, 32),
                                                 (1, 1, 3, 40), (4, 2, 33, 20)])
@pytest.mark.parametrize("all_pairs,chunk_filter", [(False, False), (True, False), (False, True), (True, True)])
def test_widths_and_multichunk_parity(P, lw, gw, threads, lanes, all_pairs, chunk_filter):
    # every word-width variant of the trigger kernel; (1, 1, 3, 40): 120
    # chunks of one group, i.e. four chunks per bit of the chunk-level table
    run_both(P, n=20_000, threads=threads, lanes=lanes, nv=300, lane_width=lw, group_width=gw,
             seed=lw * 100 + gw, rounds=2, size_lo=0, size_hi=12, all_pairs=all_pairs and lanes > lw,
             chunk_filter=chunk_filter)


def test_c3_shape_parity(P):
    run_both(P, n=150_000, threads=32, lanes=32, nv=200_000, seed=23)


@pytest.mark.parametrize("lw,gw,all_pairs,chunk_filter", [(1, 64, False, False), (1, 64, True, False),
                                                          (2, 32, False, True), (3, 8, True, True)])
def test_many_chunks_parity(P, lw, gw, all_pairs, chunk_filter):
    # hundreds of groups in one round: 1200 groups of one lane = 19 chunks of
    # 64 (group indices far past 8 bits, the group table read from global
    # memory), threads spanning chunks, with and without the chunk filter
    run_both(P, n=6000, threads=4, lanes=300, nv=400, seed=13, lane_width=lw, group_width=gw,
             size_lo=2, size_hi=12, all_pairs=all_pairs, chunk_filter=chunk_filter)


def test_large_variable_range_parity(P):
    # 3M variables: table rows of 3M entries (lane table ~0.8 GB per slot),
    # variable ids past 2^21 in every index computation
    res = run_both(P, n=20_000, threads=2, lanes=32, nv=3_000_000, seed=29, size_lo=1, size_hi=6)
    assert res.reports > 0


def test_long_clauses_parity(P):
    # clauses far longer than the prefetched rows (and past the 58 ordered positions)
    run_both(P, n=3000, threads=4, lanes=32, nv=2000, seed=9, size_lo=100, size_hi=400)
    run_both(P, n=3000, threads=4, lanes=64, nv=2000, seed=9, size_lo=100, size_hi=400, group_width=1,
             all_pairs=True)


def test_non_consecutive_thread_groups_rejected(P):
    # the one-report-per-(clause, thread) rule needs a thread's groups to be
    # consecutive, as run_round's grouping makes them (engine.py:390-399)
    from paper_2012_03119_b200.native import NativeEngine
    e = NativeEngine(10)
    with pytest.raises(ValueError):
        e.prepare(np.array([1, 1, 1], np.int32), np.array([0, 1, 0], np.int32))
    e.prepare(np.array([1, 1, 1], np.int32), np.array([0, 0, 1], np.int32))
    e.close()


def test_reduce_and_remove_parity(P):
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    rng = np.random.default_rng(3)
    nv = 500
    buckets = W.clause_buckets(30_000, nv, rng, 1, 20)
    flat, offs, ids = W.flatten(buckets)
    org = np.zeros(len(ids), np.int32)
    dev = NativeEngine(nv)
    dev.add_clauses(flat, offs, ids, org, 1.0)
    ora = O.OracleStore()
    k = 0
    for s, arr in buckets.items():
        for row in arr:
            ora.insert(row.tolist(), int(ids[k]), 0, 1.0)
            k += 1
    inc = 1.0
    for r in range(3):  # create activity diversity with ties
        snaps = W.snapshots(2, 32, nv, rng)
        gl, gt = W.groups_for(2, 32)
        dev.stage(snaps)
        dev.round(gl, gt, inc)
        ora.test_round(nv, snaps, gl, gt, 32, 32, inc)
        inc *= 2
    got = dev.reduce(20_000, 9_000)
    n, want = ora.reduce(20_000, 9_000)
    assert len(got) == n == 9_000 and np.array_equal(got, np.sort(want))  # ids ascending
    # ties at the threshold: equal activities are ordered by id (engine.py:488-489)
    got2 = dev.reduce(10 ** 9, 1234)
    n2, want2 = ora.reduce(10 ** 9, 1234)
    assert np.array_equal(got2, np.sort(want2))
    dels = rng.choice(ids, 2000, replace=False)
    assert dev.remove(dels) == ora.remove(dels.tolist())
    dev.scale(1e-100)
    ora.scale(1e-100)
    for (s, lits, i1, o1, a1), (s2, n2, lits2, i2, o2, a2) in zip(dev.buckets(), ora.buckets()):
        assert np.array_equal(lits, lits2) and np.array_equal(i1, i2)
        assert np.array_equal(a1.view(np.uint64), a2.view(np.uint64))
    # the store keeps testing correctly after compaction
    snaps = W.snapshots(2, 32, nv, rng)
    gl, gt = W.groups_for(2, 32)
    dev.stage(snaps)
    res = dev.round(gl, gt, 3.0)
    recs, ctr = ora.test_round(nv, snaps, gl, gt, 32, 32, 3.0)
    assert res.reports == len(recs) and res.lane_triggers == ctr["lane_triggers"]


@pytest.mark.parametrize("gw", [32, 2])
def test_report_buffer_overflow_replay(P, gw):
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    rng = np.random.default_rng(11)
    nv = 50
    buckets = W.clause_buckets(50_000, nv, rng, 1, 3)
    flat, offs, ids = W.flatten(buckets)
    dev = NativeEngine(nv, 32, gw, report_capacity=16)
    dev.add_clauses(flat, offs, ids)
    snaps = W.snapshots(4, 32, nv, rng)
    gl, gt = W.groups_for(4, 32)
    dev.stage(snaps)
    res = dev.round(gl, gt, 1.0)
    assert res.reruns == 1 and res.reports > 16
    ora = O.OracleStore()
    ora.insert_flat(flat, offs, ids)
    orecs, octr = ora.test_round(nv, snaps, gl, gt, 32, gw, 1.0)
    recs = dev.fetch(res.reports)
    assert sorted(zip(recs["engine_id"].tolist(), recs["group"].tolist(), recs["lane_mask"].tolist())) == \
        sorted(zip(orecs["engine_id"].tolist(), orecs["group"].tolist(), orecs["lane_mask"].tolist()))
    acts_dev = np.concatenate([b[4] for b in dev.buckets()])
    acts_ora = np.concatenate([b[5] for b in ora.buckets()])
    assert np.array_equal(acts_dev.view(np.uint64), acts_ora.view(np.uint64))


def _tables(eng):
    import torch
    ptr_, nbytes = eng.tables()

    class _CAI:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr_, False), "version": 3}
    eng.sync()
    return torch.as_tensor(_CAI(), device="cuda").cpu().numpy().copy()


def _defined_tables(raw, nv, lw, gw, gl, chunk_filter=False):
    """The written entries of the round tables (tsg_engine.cu layout: per chunk
    agg[V+2] then lane[G][vstride], each region 256-byte aligned)."""
    def up(x, m):
        return (x + m - 1) // m * m
    aeb = 32 if gw > 32 else 16
    leb = 16 if lw > 32 else 8
    vstride = up(nv + 2, 4)
    stride = up((nv + 2) * aeb, 256) + up(vstride * gw * leb, 256)  # every chunk's tables, uniform stride
    parts = []
    for c in range(0, len(gl), gw):
        G = min(gw, len(gl) - c)
        off = c // gw * stride
        parts.append(raw[off:off + (nv + 2) * aeb].reshape(nv + 2, aeb)[:, :3 * aeb // 4])  # t, f, u
        off += up((nv + 2) * aeb, 256)
        lane = raw[off:off + vstride * G * leb].reshape(G, vstride, leb)[:, :nv + 2]
        parts.append(lane.reshape(-1))
    if chunk_filter and len(gl) > gw:  # the chunk-level aggregate after the chunks: t, f, u of every variable
        off = (len(gl) + gw - 1) // gw * stride
        parts.append(raw[off:off + (nv + 2) * 16].reshape(nv + 2, 16)[:, :12])
    return np.concatenate([x.reshape(-1) for x in parts])


@pytest.mark.parametrize("lw,gw,threads,lanes,nv", [(32, 32, 3, 40, 1000), (64, 64, 2, 100, 333),
                                                    (64, 8, 5, 70, 4095), (7, 3, 4, 20, 31), (32, 32, 32, 32, 20_000)])
@pytest.mark.parametrize("chunk_filter", [False, True])
def test_packed_rows_encode_identically(P, lw, gw, threads, lanes, nv, chunk_filter):
    # snapshot ingress in 2-bit packed rows: the packed encoder must build
    # byte-identical lane/aggregate tables, and the round identical results
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine, pack_rows
    rng = np.random.default_rng(nv)
    buckets = W.clause_buckets(5000, nv, rng, 1, 10)
    flat, offs, ids = W.flatten(buckets)
    snaps = W.snapshots(threads, lanes, nv, rng)
    snaps[:, 0] = rng.integers(-1, 2, snaps.shape[0])  # slot 0 must be ignored
    snaps[::7, 5 % (nv + 1)] = 9                       # non-{1,-1,0} values read as False
    gl, gt = W.groups_for(threads, lanes, lw)
    out = []
    for packed in (False, True):
        e = NativeEngine(nv, lw, gw, chunk_filter=chunk_filter)
        e.add_clauses(flat, offs, ids)
        if packed:
            e.stage_packed(pack_rows(snaps, nv, threads=2))
        else:
            e.stage(snaps)
        e.prepare(gl, gt)
        e.encode()
        tab = _defined_tables(_tables(e), nv, lw, gw, gl, chunk_filter)
        res = e.test(1.0)
        recs = np.sort(e.fetch(res.reports), order=["engine_id", "group"])
        out.append((tab, res.lane_triggers, res.aggregate_tests_negative, recs))
        e.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1:3] == out[1][1:3]
    assert np.array_equal(out[0][3], out[1][3])


@pytest.mark.parametrize("nv", [1000, 333, 4095, 31])
def test_mixed_staging_encodes_identically(P, nv):
    # rows partly packed on the host and partly copied as int8 and packed on
    # the device (tsg_stage_packed_mixed): byte-identical tables to all-packed
    # staging at every split, and identical round results
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine, pack_rows
    rng = np.random.default_rng(nv + 1)
    buckets = W.clause_buckets(4000, nv, rng, 1, 10)
    flat, offs, ids = W.flatten(buckets)
    snaps = W.snapshots(3, 40, nv, rng)
    snaps[:, 0] = rng.integers(-1, 2, snaps.shape[0])  # slot 0 must be ignored
    snaps[::7, 5 % (nv + 1)] = 9                       # non-{1,-1,0} values read as False
    gl, gt = W.groups_for(3, 40, 32)
    packed_all = pack_rows(snaps, nv)
    want = None
    for split in (snaps.shape[0], 0, 1, 57, snaps.shape[0] - 1):
        e = NativeEngine(nv, 32, 32)
        e.add_clauses(flat, offs, ids)
        if split == snaps.shape[0]:
            e.stage_packed(packed_all)
        else:
            e.stage_packed_mixed(packed_all[:split], snaps[split:])
        e.prepare(gl, gt)
        e.encode()
        tab = _defined_tables(_tables(e), nv, 32, 32, gl)
        res = e.test(1.0)
        got = (tab, res.lane_triggers, np.sort(e.fetch(res.reports), order=["engine_id", "group"]))
        e.close()
        if want is None:
            want = got
        else:
            assert np.array_equal(got[0], want[0]), split
            assert got[1] == want[1] and np.array_equal(got[2], want[2]), split


def test_async_report_egress_double_buffered(P):
    # round k's records copy out on the egress stream while round k+1 runs;
    # every round's records must equal a synchronous fetch of the same round
    import torch
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    from paper_2012_03119_b200._lib import REPORT_DTYPE
    rng = np.random.default_rng(5)
    nv = 3000
    buckets = W.clause_buckets(40_000, nv, rng, 1, 8)
    flat, offs, ids = W.flatten(buckets)
    rounds = [W.snapshots(4, 32, nv, rng) for _ in range(5)]
    gl, gt = W.groups_for(4, 32)
    a, b = NativeEngine(nv, report_capacity=1024), NativeEngine(nv)
    a.add_clauses(flat, offs, ids)
    b.add_clauses(flat, offs, ids)
    cap = 1 << 20
    bufs = [torch.empty(cap * 16, dtype=torch.uint8).pin_memory().numpy().view(REPORT_DTYPE) for _ in range(2)]
    got, want = [], []
    for k, snaps in enumerate(rounds):
        a.stage(snaps)
        ra = a.round(gl, gt, 1.0)
        n = a.fetch_async(bufs[k % 2])
        assert n == ra.reports
        b.stage(snaps)
        rb = b.round(gl, gt, 1.0)
        want.append(np.sort(b.fetch_raw(rb.reports), order=["key"]))
        if k % 2 == 1:  # both buffers in flight: wait, then read them
            a.wait()
            got.append(np.sort(bufs[0][:prev_n].copy(), order=["key"]))
            got.append(np.sort(bufs[1][:n].copy(), order=["key"]))
        prev_n = n
    assert len(got) == 4
    for g, w in zip(got, want[:4]):
        assert np.array_equal(g, w)
    a.close()
    b.close()


def test_c3_full_size_parity(P):
    # the benchmark's own workload (bench.py C3: 10M clauses x 1024 assignments,
    # 200k vars, same seeds) through the benchmark's ingress path (packed rows):
    # every record, counter and fp64 activity bit-exact against the oracle
    import os
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine, pack_rows
    cfg = W.CONFIGS["C3"]
    rng = np.random.default_rng(cfg.seed)
    buckets = W.clause_buckets(cfg.n_clauses, cfg.num_vars, rng, cfg.size_lo, cfg.size_hi)
    flat, offs, ids = W.flatten(buckets)
    snaps = W.snapshots(cfg.threads, cfg.lanes, cfg.num_vars, np.random.default_rng(cfg.seed + 999))
    gl, gt = W.groups_for(cfg.threads, cfg.lanes)
    dev = NativeEngine(cfg.num_vars, report_capacity=8 << 20)
    dev.add_clauses(flat, offs, ids)
    dev.stage_packed(pack_rows(snaps, cfg.num_vars, threads=os.cpu_count() or 1))
    res = dev.round(gl, gt, 1.0)
    recs = np.sort(dev.fetch(res.reports), order=["engine_id", "group"])
    ora = O.OracleStore()
    ora.insert_flat(flat, offs, ids)
    del flat
    orecs, octr = ora.test_round(cfg.num_vars, snaps, gl, gt, 32, 32, 1.0, nthreads=os.cpu_count() or 1)
    assert res.reports == len(orecs) == len(recs) > 1_000_000
    o = np.zeros(len(orecs), recs.dtype)
    for f in ("engine_id", "group", "lane_mask"):
        o[f] = orecs[f]
    o = np.sort(o, order=["engine_id", "group"])
    for f in ("engine_id", "group", "lane_mask"):
        assert np.array_equal(recs[f], o[f]), f
    for k in ("clauses_tested", "aggregate_tests", "aggregate_tests_negative", "lane_tests", "lane_triggers"):
        assert getattr(res, k) == octr[k], k
    for (s, lits, i1, o1, a1), (s2, n2, lits2, i2, o2, a2) in zip(dev.buckets(), ora.buckets()):
        assert s == s2 and np.array_equal(i1, i2)
        assert np.array_equal(a1.view(np.uint64), a2.view(np.uint64))
    dev.close()


@pytest.mark.parametrize("cap", [1 << 20, 64])  # 64: every round overflows and replays with the next in flight
@pytest.mark.parametrize("gw", [32, 1])  # gw 1: multi-chunk rounds (chunk-level aggregate)
# pinned: rows copy in asynchronously on the ingress stream; rec 8: the kernel writes 8-byte records
@pytest.mark.parametrize("pinned,rec", [(False, 16), (True, 16), (False, 8), (True, 8)])
def test_async_rounds_match_sync_rounds(P, cap, gw, pinned, rec):
    # two rounds in flight: launch(k-1), launch(k), collect(k-1) ...: identical
    # figures, records and activities to synchronous rounds, overflow replays included
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine, pack_rows
    rng = np.random.default_rng(17)
    nv = 2000
    buckets = W.clause_buckets(30_000, nv, rng, 1, 9)
    flat, offs, ids = W.flatten(buckets)
    rounds = []
    for k in range(5):
        threads = 2 + k % 3
        snaps = W.snapshots(threads, 32, nv, rng)
        rounds.append((snaps, *W.groups_for(threads, 32)))
    a = NativeEngine(nv, 32, gw, report_capacity=cap)
    b = NativeEngine(nv, 32, gw)
    if rec == 8:
        a.set_record_bytes(8)
    a.add_clauses(flat, offs, ids)
    b.add_clauses(flat, offs, ids)
    fields = ("reports", "clauses_tested", "aggregate_tests", "aggregate_tests_negative", "lane_tests",
              "lane_triggers")
    want = []
    for k, (snaps, gl, gt) in enumerate(rounds):
        b.stage(snaps)
        r = b.round(gl, gt, 1.0 + k)
        want.append(([getattr(r, f) for f in fields], np.sort(b.fetch(r.reports), order=["engine_id", "group"])))
    got, keep = [], []

    def take():
        r = a.collect()  # the oldest launched round
        got.append(([getattr(r, f) for f in fields], np.sort(a.fetch(r.reports), order=["engine_id", "group"])))

    for k, (snaps, gl, gt) in enumerate(rounds):  # two rounds in flight
        if k >= 2:
            take()  # round k-2 owns the table slot round k encodes into
        rows = pack_rows(snaps, nv)
        if pinned:  # one pinned buffer per round: unchanged until its round is collected
            import torch
            buf = torch.empty(rows.shape, dtype=torch.int64).pin_memory()
            keep.append(buf)
            rows = np.copyto(buf.numpy().view(np.uint64), rows) or buf.numpy().view(np.uint64)
        a.stage_packed(rows)
        a.prepare(gl, gt)
        a.encode()
        a.launch(1.0 + k)
    take()
    take()
    for (gf, gr), (wf, wr) in zip(got, want):
        assert gf == wf
        assert np.array_equal(gr, wr)
    for x, y in zip(a.buckets(), b.buckets()):
        assert np.array_equal(x[4].view(np.uint64), y[4].view(np.uint64))
    with pytest.raises(ValueError):  # at most two rounds in flight
        a.prepare(*rounds[0][1:])
        a.encode()
        a.launch(1.0)
        a.launch(1.0)
        a.launch(1.0)
    a.close()
    b.close()


def test_abi_error_paths(P):
    # errors surface as the reference's exception types (bitpack.py:30-36,
    # 92-103; engine.py:64-74), never as silent fallbacks
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine, pack_rows, packed_words
    from paper_2012_03119_b200._lib import CapacityError
    nv = 1000
    e = NativeEngine(nv, 8, 4)
    flat, offs, ids = W.flatten(W.clause_buckets(500, nv, np.random.default_rng(1), 1, 5))
    e.add_clauses(flat, offs, ids)
    snaps = W.snapshots(2, 8, nv, np.random.default_rng(2))
    with pytest.raises(ValueError):  # packed pitch shorter than a row
        e.stage_packed(np.ascontiguousarray(pack_rows(snaps, nv)[:, :packed_words(nv) - 4]))
    with pytest.raises(CapacityError):  # more lanes than lane_width
        e.prepare(np.array([9], np.int32), np.array([0], np.int32))
    with pytest.raises(ValueError):  # groups need more rows than staged
        e.stage(snaps[:4])
        e.prepare(*W.groups_for(2, 8, 8))
        e.encode()
    e.stage(snaps)
    e.prepare(*W.groups_for(2, 8, 8))
    e.encode()
    e.launch(1.0)
    with pytest.raises(ValueError):  # the store is frozen while a round is in flight
        e.add_clauses(flat[:3], np.array([0, 3], np.int64), np.array([10 ** 6], np.int64))
    with pytest.raises(ValueError):
        e.remove(np.array([0]))
    r = e.collect()
    assert r.reports == len(e.fetch(r.reports))
    with pytest.raises(ValueError):  # nothing in flight
        e.collect()
    e.close()


def test_twelve_byte_egress_records(P):
    # 12- and 8-byte egress records carry the same (engine id, group, lane
    # mask) as the 16-byte tsg_report, sync and async; lane_width 64 refuses them
    from paper_2012_03119_b200 import reports as R
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    rng = np.random.default_rng(21)
    nv = 2000
    flat, offs, ids = W.flatten(W.clause_buckets(30_000, nv, rng, 1, 8))
    snaps = W.snapshots(3, 32, nv, rng)
    gl, gt = W.groups_for(3, 32)
    out = []
    for nbytes in (16, 12, 8):
        e = NativeEngine(nv)
        e.set_record_bytes(nbytes)
        e.add_clauses(flat, offs, ids)
        e.stage(snaps)
        r = e.round(gl, gt, 1.0)
        sync = np.sort(R.decode(e.fetch_raw(r.reports)), order=["engine_id", "group"])
        buf = np.zeros(r.reports, {16: R.RECORD_DTYPE, 12: R.RECORD12_DTYPE, 8: R.RECORD8_DTYPE}[nbytes])
        assert e.fetch_async(buf) == r.reports
        e.wait()
        out.append((sync, np.sort(R.decode(buf), order=["engine_id", "group"])))
        e.close()
    assert len(out[0][0]) > 100
    for a in out:
        for b in out:
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    w = NativeEngine(nv, 64, 32)
    for nbytes in (12, 8):
        with pytest.raises(ValueError):
            w.set_record_bytes(nbytes)
    w.close()
    # 8-byte records refuse engine ids >= 2^27 and rounds of more than 32 groups
    from paper_2012_03119_b200._lib import CapacityError
    for big_id, threads in ((True, 3), (False, 33)):
        e = NativeEngine(nv)
        e.set_record_bytes(8)
        e.add_clauses(flat, offs, ids + ((1 << 27) if big_id else 0))
        sn = W.snapshots(threads, 32, nv, rng)
        e.stage(sn)
        r = e.round(*W.groups_for(threads, 32), 1.0)
        assert r.reports > 0
        with pytest.raises(CapacityError):
            e.fetch_raw(r.reports)
        e.close()


def test_get_clauses_and_counters(P):
    # tsg_get_clauses returns stored clauses by engine id in their original
    # literal order (engine.py:165-169) despite the pivot / polarity layout,
    # None once removed; tsg_counters accumulates the round figures
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    rng = np.random.default_rng(5)
    nv = 3000
    flat, offs, ids = W.flatten(W.clause_buckets(50_000, nv, rng, 0, 30))
    e = NativeEngine(nv)
    e.add_clauses(flat, offs, ids)
    want = {int(ids[i]): tuple(flat[offs[i]:offs[i + 1]].tolist()) for i in range(len(ids))}
    pick = rng.choice(ids, 2000, replace=False)
    q = np.concatenate([pick, [ids.max() + 1, -5], pick[:3]])  # missing ids and repeats
    got = e.get_clauses(q)
    assert got[:2000] == [want[int(i)] for i in pick]
    assert got[2000:2002] == [None, None] and got[2002:] == [want[int(i)] for i in pick[:3]]
    figs = []
    for k in range(3):
        e.stage(W.snapshots(2, 32, nv, rng))
        r = e.round(*W.groups_for(2, 32), 1.0)
        figs.append(r)
    gone = e.remove(pick[:100])
    assert gone == 100 and e.get_clauses(pick[:100]) == [None] * 100
    assert e.get_clauses(pick[100:200]) == [want[int(i)] for i in pick[100:200]]
    c = e.counters()
    assert c["rounds"] == 3 and c["clauses_added"] == len(ids) and c["clauses_deleted"] == 100
    for f in ("reports", "clauses_tested", "aggregate_tests", "aggregate_tests_negative", "lane_tests",
              "lane_triggers"):
        assert c[f] == sum(getattr(r, f) for r in figs), f
    e.close()


def test_timing_sampling(P):
    # tsg_set_timing(n): only rounds whose launch sequence is a multiple of n
    # carry event timings; the others report -1 (figures unaffected)
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    rng = np.random.default_rng(9)
    nv = 2000
    flat, offs, ids = W.flatten(W.clause_buckets(20_000, nv, rng, 1, 9))
    e = NativeEngine(nv, timing=True)
    e.add_clauses(flat, offs, ids)
    e.set_timing(2)
    snaps = W.snapshots(2, 32, nv, rng)
    gl, gt = W.groups_for(2, 32)
    got = []
    for _ in range(4):
        e.stage(snaps)
        got.append(e.round(gl, gt, 1.0))
    assert [r.test_ms >= 0 for r in got] == [False, True, False, True]
    assert all((r.encode_ms >= 0) == (r.test_ms >= 0) for r in got)
    assert len({r.reports for r in got}) == 1
    e.set_timing(0)
    e.stage(snaps)
    assert e.round(gl, gt, 1.0).test_ms == -1
    with pytest.raises(ValueError):
        e.set_timing(-1)
    e.close()


def test_replay_with_threads_spanning_chunks(P):
    # overflow replays of rounds whose threads span chunk boundaries (the
    # one-report-per-(clause, thread) rule across chunks), engine after
    # engine in one process -- every run must match the oracle
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    nv = 300
    for seed in (1, 5):
        rng = np.random.default_rng(seed)
        buckets = W.clause_buckets(60000, nv, rng, 0, 12)
        flat, offs, ids = W.flatten(buckets)
        snaps = W.snapshots(3, 58, nv, rng)
        gl, gt = W.groups_for(3, 58, 16)  # 4 groups per thread, 3 per chunk
        st = O.OracleStore()
        st.insert_flat(flat, offs, ids)
        want, _ = st.test_round(nv, snaps, gl, gt, 16, 3, 1.0, nthreads=8)
        for cap in (0, 64, 0, 64):
            e = NativeEngine(nv, 16, 3, report_capacity=cap)
            e.add_clauses(flat, offs, ids)
            e.stage(snaps)
            r = e.round(gl, gt, 1.0)
            assert r.reports == len(want)
            recs = W.in_reference_order(e.fetch(r.reports), offs, ids, buckets, 3)
            for f in ("engine_id", "lane_mask", "group"):
                assert np.array_equal(recs[f], want[f]), f
            e.close()


@pytest.mark.parametrize("all_pairs", [False, True])
def test_repeated_literals_and_tautologies_parity(P, all_pairs):
    # the reference accepts any literal list (engine.py:305-317): repeated
    # literals and x or -x in one clause change nothing in its recurrences,
    # and the store keeps them; drawn from 40 variables so both are common
    import os
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    rng = np.random.default_rng(23)
    nv, threads, lanes = 40, 3, 32
    sizes = rng.integers(1, 9, 4000)
    buckets = {}
    for s in np.unique(sizes):  # bucket creation order = first-seen size order (flatten keeps dict order)
        k = int((sizes == s).sum())
        v = rng.integers(1, nv + 1, (k, int(s)))
        sg = rng.integers(0, 2, (k, int(s))) * 2 - 1
        buckets[int(s)] = (v * sg).astype(np.int32)
    flat, offs, ids = W.flatten(buckets)
    lits = [flat[offs[i]:offs[i + 1]] for i in range(len(ids))]
    assert any(len(set(np.abs(c).tolist())) < len(c) for c in lits)  # repeats and tautologies present
    assert any(set(c.tolist()) & set((-c).tolist()) for c in lits)
    dev = NativeEngine(nv, 32, 32, report_capacity=1 << 16)
    if all_pairs:
        dev.set_all_pairs(True)
    dev.add_clauses(flat, offs, ids)
    ora = O.OracleStore()
    ora.insert_flat(flat, offs, ids)
    for r in range(3):
        snaps = W.snapshots(threads, lanes, nv, rng)
        gl, gt = W.groups_for(threads, lanes, 32)
        dev.stage(snaps)
        res = dev.round(gl, gt, 1.0 + r)
        recs = W.in_reference_order(dev.fetch(res.reports), offs, ids, buckets, 32)
        ogt = np.arange(len(gl), dtype=np.int32) if all_pairs else gt
        orecs, octr = ora.test_round(nv, snaps, gl, ogt, 32, 32, 1.0 + r, nthreads=os.cpu_count() or 8)
        assert len(recs) == len(orecs) > 0
        for f in ("engine_id", "lane_mask", "group"):
            assert np.array_equal(recs[f], orecs[f]), f
        assert res.lane_triggers == octr["lane_triggers"]
        assert res.aggregate_tests_negative == octr["aggregate_tests_negative"]
    for d, o in zip(dev.buckets(), ora.buckets()):
        assert np.array_equal(d[1], o[2])  # the stored literals, as given (repeats and all)
        assert np.array_equal(d[4].view(np.uint64), o[5].view(np.uint64))
    dev.close()
