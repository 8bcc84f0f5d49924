"""C5 at the real instance size with trace on: every traced round of the
GPU engine checked against the CPU oracle for that round's store and
snapshots (sound and complete reports), plus the run's exchange figures.

    python tools/c5_verify.py [n=20000] [threads=8] [seconds=20]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2012_03119_b200 import exchange as X  # noqa: E402
from oracle import oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 8
secs = float(sys.argv[3]) if len(sys.argv) > 3 else 20.0
formula = X.random_3cnf(n, 4.26, 20121 + 5)
engines = []
ans = X.run(formula, threads=threads, timeout=secs, seed=5, gpu=True, trace=True, keep=engines)
eng = engines[0]
lw, gw = eng.config.lane_width, eng.config.group_width
checked = rounds_with = reports = snaps = 0
for tr in eng.trace:
    if not tr.snapshots:
        continue
    rounds_with += 1
    by = {}
    for tid, v in tr.snapshots:
        by.setdefault(tid, []).append(v)
    rows, gl, gt = [], [], []
    for tid in sorted(by):
        s = by[tid]
        for i in range(0, len(s), lw):
            rows.extend(s[i:i + lw])
            gl.append(len(s[i:i + lw]))
            gt.append(tid)
    st = O.OracleStore()
    for eid, lits in tr.store:
        st.insert(list(lits), eid, 0, 1.0)
    recs, _ = st.test_round(n, np.stack(rows), gl, gt, lw, gw, 1.0, nthreads=8)
    want = sorted((gt[int(r["group"])], int(r["engine_id"]), int(r["lane_mask"])) for r in recs)
    got = sorted((r.destination, r.engine_id, r.lane_mask) for r in tr.reports)
    assert got == want, (rounds_with, len(got), len(want))
    checked += 1
    reports += len(got)
    snaps += len(rows)
print(json.dumps({"instance": f"random 3-SAT n={n} (seed {20121 + 5})", "threads": threads, "seconds": secs,
                  "rounds_checked": checked, "snapshots": snaps, "reports": reports,
                  "summary": X.summary(ans)}))
for e in engines:
    e.close()
