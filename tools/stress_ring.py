"""Randomized stress of the host report ring (tsg_ring_*): two engines on the
same store -- A writes its records into the ring (random capacity 128..64 K,
1-4 drainer threads, rounds launched two in flight), B into the device
buffer -- over random rounds; every round's record set must be identical.

    python tools/stress_ring.py [seconds=120] > gpurun_out/stress_ring.txt
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_03119_b200 import reports  # noqa: E402
from paper_2012_03119_b200 import workload as W  # noqa: E402
from paper_2012_03119_b200.native import NativeEngine, RingDrainer, pack_rows  # noqa: E402


def as_set(dec):
    return set(zip(dec["engine_id"].tolist(), dec["group"].tolist(), dec["lane_mask"].tolist()))


def main(secs):
    rng = np.random.default_rng(int(time.time()))
    t_end = time.time() + secs
    n_rounds = n_recs = n_cfg = 0
    while time.time() < t_end:
        nv = int(rng.integers(50, 5000))
        n = int(rng.integers(1000, 80_000))
        lw = int(rng.choice([8, 16, 32]))
        gw = int(rng.choice([2, 8, 32]))
        all_pairs = bool(rng.integers(0, 2))
        buckets = W.clause_buckets(n, nv, rng, 1, int(rng.integers(3, 20)))
        flat, offs, ids = W.flatten(buckets)
        a = NativeEngine(nv, lw, gw, report_capacity=1 << 12)
        b = NativeEngine(nv, lw, gw, report_capacity=1 << 12)
        for e in (a, b):
            e.set_all_pairs(all_pairs)
            e.add_clauses(flat, offs, ids)
        cap = int(rng.choice([128, 1024, 1 << 16]))
        a.ring_open(capacity=cap, wait_ms=20_000)
        dr = RingDrainer(a, threads=int(rng.integers(1, 5)), batch=int(rng.choice([64, 4096])))
        try:
            pending = []
            for k in range(int(rng.integers(3, 12))):
                threads = int(rng.integers(1, 6))
                lanes = int(rng.integers(1, 3 * lw))
                snaps = W.snapshots(threads, lanes, nv, rng)
                gl, gt = W.groups_for(threads, lanes, lw)
                b.stage(snaps)
                rb = b.round(gl, gt, 1.0)
                want = as_set(b.fetch(rb.reports))
                if len(pending) == 2:  # two rounds in flight on A
                    r0, w0 = pending.pop(0)
                    got = a.collect()
                    assert got.reports == r0, (got.reports, r0)
                    recs = reports.decode(dr.take(got.reports))
                    assert len(recs) == got.reports and as_set(recs) == w0
                    n_recs += got.reports
                a.stage_packed(pack_rows(snaps, nv))
                a.prepare(gl, gt)
                a.encode()
                a.launch(1.0)
                pending.append((rb.reports, want))
                n_rounds += 1
            while pending:
                r0, w0 = pending.pop(0)
                got = a.collect()
                assert got.reports == r0
                recs = reports.decode(dr.take(got.reports))
                assert as_set(recs) == w0
                n_recs += got.reports
            exp, con, failed = a.ring_status()
            assert exp == con and not failed, (exp, con, failed)
        finally:
            dr.close()
            a.ring_close()
            a.close()
            b.close()
        n_cfg += 1
    print(f"stress_ring: {n_cfg} configurations, {n_rounds} rounds, {n_recs} ring records, all identical "
          f"to the device-buffer path", flush=True)


if __name__ == "__main__":
    main(float(sys.argv[1]) if len(sys.argv) > 1 else 120.0)
