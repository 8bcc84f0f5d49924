"""C4 streaming measurement: the Engine API (the
reference's surface) under a steady clause/assignment stream.

Per round: `adds` new clauses (sizes U[2,30]) from the 32 producer threads,
`dels` explicit deletes of live ids, 32 threads x 64 snapshots (queue cap
64 -> 2048 assignments, 2 chunks of 32 groups), store capped at
`max_clauses` (reduce_store when full), reports drained by every thread.
Metric: the reference's own clauses_tested_per_second = lane_tests /
busy_seconds (instrumentation.py:248-250), plus rounds/s and the share of
round time spent outside the GPU.

    python tools/stream_bench.py [max_clauses=1000000] [num_vars=50000] [rounds=20]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_03119_b200 as P  # noqa: E402
from paper_2012_03119_b200 import workload as W  # noqa: E402

max_clauses = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 50_000
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 20
threads, cap, adds, dels = 32, 64, 20_000, 5_000
rng = np.random.default_rng(20121 + 4)
eng = P.Engine(nv, threads, P.EngineConfig(max_clauses=max_clauses, assignment_queue_capacity=cap, timing=True))
# fill to capacity
for s, arr in W.clause_buckets(max_clauses, nv, rng).items():
    for row in arr:
        eng.add_clause(tuple(int(x) for x in row), origin=0)
eng.run_round()
pool = [W.snapshots(1, cap, nv, rng) for _ in range(4)]  # snapshot rows reused across rounds
live_lo = 0
t_sub = t_round = t_int = 0.0
eng.counters["busy_seconds"] = 0.0
eng.counters["lane_tests"] = 0
n_rep = 0
prof = None
if os.environ.get("TSG_PROFILE"):
    import cProfile
    prof = cProfile.Profile()
for r in range(rounds):
    if prof is not None and r == 1:
        prof.enable()
    new = W.clause_buckets(adds, nv, rng)
    for s, arr in new.items():
        for row in arr:
            eng.add_clause(tuple(int(x) for x in row), origin=int(rng.integers(0, threads)))
    eng.remove_clauses(rng.integers(0, eng._next_id, dels))
    t0 = time.perf_counter()
    for t in range(threads):
        rows = pool[(r + t) % len(pool)]
        for i in range(cap):
            eng.submit_assignment(P.AssignmentSnapshot(t, rows[i], i))
    t_sub += time.perf_counter() - t0
    t0 = time.perf_counter()
    eng._integrate_exports()  # (run_round would do it first; timed apart here)
    t1 = time.perf_counter()
    eng.run_round()
    t2 = time.perf_counter()
    t_round += t2 - t0
    t_int += t1 - t0
    for t in range(threads):
        n_rep += len(eng.drain_reports(t))
if prof is not None:
    prof.disable()
    import pstats
    pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(25)
c = eng.raw_counters()
print(json.dumps({
    "config": f"C4: store capped at {max_clauses}, {nv} vars, {threads} threads x {cap} snapshots/round, "
              f"+{adds} adds, {dels} deletes per round",
    "rounds": rounds, "clauses_tested_per_second": c["lane_tests"] / c["busy_seconds"],
    "round_ms": t_round / rounds * 1e3, "integrate_ms": t_int / rounds * 1e3,
    "submit_ms_per_round": t_sub / rounds * 1e3,
    "reports_per_round": n_rep / rounds, "reduces": c["reduces"], "store_size": c["store_size"],
    "gpu_ms_per_round": (eng.last_round.encode_ms + eng.last_round.test_ms) if eng.config.timing else None,
}))
