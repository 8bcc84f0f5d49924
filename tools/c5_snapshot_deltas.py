"""SURVEY.md §8(f)1 analysis (build container only: imports the reference from
/root/reference): capture the snapshots the reference's CDCL threads submit
on the C5 instance (random 3-SAT, n = 20000, ratio 4.26, 8 threads, the
reference engine on the CPU) and measure how a thread's consecutive
snapshots differ -- the size a delta / sparse ingress format would have
against the 2-bit packed rows.

    python tools/c5_snapshot_deltas.py [seconds=40]
"""
import os
import sys

import numpy as np

sys.path.insert(0, '/root/reference/pkg/src')
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import triggersat.engine as RE  # noqa: E402
import triggersat.orchestrator as orch  # noqa: E402
from paper_2012_03119_b200 import exchange as X  # noqa: E402
snaps = []
orig = RE.Engine.submit_assignment
def sub(self, s):
    if len(snaps) < 20000:
        snaps.append((s.thread_id, np.array(s.values, dtype=np.int8)))
    return orig(self, s)
RE.Engine.submit_assignment = sub
f = X.random_3cnf(20000, 4.26, 7)
cfg = orch.RunConfig(threads=8, timeout=float(sys.argv[1]) if len(sys.argv) > 1 else 30.0, seed=7)
ans = orch.solve_parallel(f, cfg)
print("status", ans.status, "snapshots", len(snaps))
prev = {}; ch = []; asg = []; wch = []
for t, v in snaps:
    asg.append(int((v != 0).sum()))
    if t in prev:
        d = prev[t] != v
        ch.append(int(d.sum()))
        w = d[:len(d) // 32 * 32].reshape(-1, 32).any(1)
        wch.append(int(w.sum()))
    prev[t] = v
ch = np.array(ch); asg = np.array(asg); wch = np.array(wch)
V = 20000
print(f"assigned per snapshot mean {asg.mean():.0f} ({asg.mean()/V:.1%} of vars)")
print(f"changed vs previous snapshot of the thread: mean {ch.mean():.0f} median {np.median(ch):.0f} p90 {np.percentile(ch,90):.0f}")
print(f"32-var words changed: mean {wch.mean():.0f} of {V//32}")
print(f"bytes/row: packed 2-bit {(V+1+31)//32*8}, var-delta (4 B each) {4*ch.mean():.0f}, word-delta (12 B each) {12*wch.mean():.0f}")
