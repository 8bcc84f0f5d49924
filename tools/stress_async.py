"""Randomised stress of the asynchronous round machinery (diagnostics):
engine A runs rounds with up to two in flight, random report capacities,
record formats, ingress from pinned / pageable rows, and store mutations
between drained pipelines; engine B runs the same rounds synchronously with
16-byte records.  Every round's figures, records and the final store
(literals, ids, fp64 activities) must match.

    python tools/stress_async.py [seconds] [seed]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2012_03119_b200 import reports as R  # noqa: E402
from paper_2012_03119_b200 import workload as W  # noqa: E402
from paper_2012_03119_b200.native import NativeEngine, pack_rows  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 60
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
nv = 3000
FIELDS = ("reports", "clauses_tested", "aggregate_tests", "aggregate_tests_negative", "lane_tests", "lane_triggers")
t_end = time.time() + secs
n_rounds = n_cases = 0
while time.time() < t_end:
    n_cases += 1
    gw = int(rng.choice([32, 16, 8]))
    cap = int(rng.choice([0, 64, 4096]))
    rec = int(rng.choice([16, 12, 8]))
    a = NativeEngine(nv, 32, gw, report_capacity=cap)
    b = NativeEngine(nv, 32, gw)
    a.set_record_bytes(rec)
    next_id = 0
    for phase in range(int(rng.integers(2, 5))):
        # store mutation with nothing in flight
        n_add = int(rng.integers(1000, 20000))
        flat, offs, _ = W.flatten(W.clause_buckets(n_add, nv, rng, 0, 20))
        ids = np.arange(next_id, next_id + len(offs) - 1, dtype=np.int64)
        next_id += len(ids)
        a.add_clauses(flat, offs, ids)
        b.add_clauses(flat, offs, ids)
        if next_id > 100 and rng.random() < 0.5:
            dead = rng.choice(next_id, int(rng.integers(1, 500)), replace=False)
            assert a.remove(dead) == b.remove(dead)
        rounds = []
        for _ in range(int(rng.integers(1, 7))):
            threads = int(rng.integers(1, 6))
            snaps = W.snapshots(threads, 32, nv, rng)
            rounds.append((snaps, *W.groups_for(threads, 32)))
        want = []
        for k, (snaps, gl, gt) in enumerate(rounds):
            b.stage(snaps)
            r = b.round(gl, gt, 1.0 + k)
            want.append(([getattr(r, f) for f in FIELDS],
                         np.sort(R.decode(b.fetch_raw(r.reports)), order=["engine_id", "group"])))
        got, keep, inflight = [], [], 0
        depth = int(rng.integers(1, 3))

        def take():
            r = a.collect()
            got.append(([getattr(r, f) for f in FIELDS],
                        np.sort(R.decode(a.fetch_raw(r.reports)), order=["engine_id", "group"])))

        for k, (snaps, gl, gt) in enumerate(rounds):
            if inflight >= depth:
                take()
                inflight -= 1
            rows = pack_rows(snaps, nv)
            if rng.random() < 0.5:
                buf = torch.empty(rows.shape, dtype=torch.int64).pin_memory()
                keep.append(buf)
                np.copyto(buf.numpy().view(np.uint64), rows)
                rows = buf.numpy().view(np.uint64)
            a.stage_packed(rows)
            a.prepare(gl, gt)
            a.encode()
            a.launch(1.0 + k)
            inflight += 1
        while inflight:
            take()
            inflight -= 1
        for (gf, gr), (wf, wr) in zip(got, want):
            assert gf == wf, (gf, wf)
            assert np.array_equal(gr, wr)
        n_rounds += len(rounds)
    for x, y in zip(a.buckets(), b.buckets()):
        assert x[0] == y[0] and np.array_equal(x[1], y[1]) and np.array_equal(x[2], y[2])
        assert np.array_equal(x[4].view(np.uint64), y[4].view(np.uint64))
    a.close()
    b.close()
print(f"stress ok: {n_cases} engine pairs, {n_rounds} rounds, seed {seed}")
