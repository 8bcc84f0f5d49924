"""Profile the drop-in Engine's round phases at C4 (cProfile of run_round).

    python tools/api_probe.py [rounds=5]
"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_03119_b200 as P  # noqa: E402
from paper_2012_03119_b200 import workload as W  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nv, threads, per, n_store, adds, dels = 50_000, 32, 64, 1_000_000, 20_000, 5_000
rng = np.random.default_rng(5)
eng = P.Engine(nv, threads, P.EngineConfig(max_clauses=n_store, assignment_queue_capacity=per))
flat, offs, _ = W.flatten(W.clause_buckets(n_store, nv, rng))
eng.add_clauses(flat, offs)
eng.run_round()
rows = W.snapshots(threads, per, nv, rng)
prof = cProfile.Profile()
for k in range(rounds):
    for arr in W.clause_buckets(adds, nv, rng).values():
        for row in arr.tolist():
            eng.add_clause(row, origin=0)
    eng.remove_clauses(rng.integers(0, eng._next_id, dels))
    for t in range(threads):
        for i in range(per):
            eng.submit_assignment(P.AssignmentSnapshot(t, rows[t * per + i], i))
    t0 = time.perf_counter()
    if k >= 1:
        prof.enable()
    eng.run_round()
    prof.disable()
    print(f"round {k}: {1e3 * (time.perf_counter() - t0):.2f} ms  phases {eng.last_phases}", flush=True)
    for t in range(threads):
        eng.drain_reports(t)
pstats.Stats(prof).sort_stats("tottime").print_stats(15)
