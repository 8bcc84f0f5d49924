"""Replay-mismatch probe (diagnostics): lw 16, gw 3, nv 300, 60k clauses of
0-12 literals, 3 threads x 58 snapshots, forced overflow replays."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_03119_b200 import workload as W  # noqa: E402
from paper_2012_03119_b200.native import NativeEngine  # noqa: E402

bad = 0
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    rng = np.random.default_rng(seed)
    nv = 300
    flat, offs, ids = W.flatten(W.clause_buckets(60000, nv, rng, 0, 12))
    snaps = W.snapshots(3, 58, nv, rng)
    gl, gt = W.groups_for(3, 58, 16)
    for cap in (0, 64):
        e = NativeEngine(nv, 16, 3, report_capacity=cap)
        e.add_clauses(flat, offs, ids)
        e.stage(snaps)
        try:
            r = e.round(gl, gt, 1.0)
            print("seed", seed, "cap", cap, "reports", r.reports, "reruns", r.reruns)
        except Exception as exc:
            bad += 1
            print("seed", seed, "cap", cap, "FAIL", exc)
        e.close()
print("failures", bad)
