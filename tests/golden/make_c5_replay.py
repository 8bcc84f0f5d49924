"""Record C5 exchange rounds from the REFERENCE solver + engine (SURVEY.md
§8(d) C5) as replay fixtures, so the GPU Engine can be checked on real solver
snapshots without the reference installed on the GPU box.

Run in the build container only (it imports the reference from
/root/reference/pkg/src):

    python tests/golden/make_c5_replay.py

The reference's `solve_parallel` (orchestrator.py:84-198) runs a random
3-SAT instance near the threshold (oracles.py:110-118 recipe) with its CDCL
threads and its own Engine in trace mode (engine.py:113-119, 425-431).  The
generator logs every clause the engine inserts (ClauseStore.insert,
engine.py:213-219) and every round's RoundResult, and writes, per traced
round that tested snapshots:

  n_inserted   clauses inserted so far (engine ids 0..n_inserted-1 in order)
  live         engine ids in the store when the round tested (trace.store)
  snap_tid, snap_vals   the round's snapshots per thread, FIFO order
  rep_dest, rep_eid, rep_mask   the reports in emission order
  result       reports_emitted, clauses_tested, assignments_consumed,
               aggregate_tests_negative

Outputs: tests/golden/c5_replay_<name>.npz (compressed, committed).
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from triggersat import engine as E  # noqa: E402
from triggersat import orchestrator as O  # noqa: E402
from triggersat.core import Formula  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# name: (num_vars, ratio, formula seed, threads, lane_width, group_width, timeout, max rounds)
CASES = {
    "w32": (150, 4.26, 2, 4, 32, 32, 60.0, 40),
    # narrow words: multi-chunk rounds, threads spanning chunks (the
    # chunk-level aggregate and the cross-chunk report rule)
    "w8x2": (150, 4.26, 2, 4, 8, 2, 60.0, 40),
}


def random_3cnf(n, ratio, seed):
    """oracles.py:110-118's recipe: m = round(ratio * n) clauses of 3 distinct variables."""
    rng = np.random.default_rng(seed)
    m = int(round(ratio * n))
    clauses = []
    for _ in range(m):
        vs = rng.choice(n, 3, replace=False) + 1
        sg = rng.integers(0, 2, 3) * 2 - 1
        clauses.append([int(v * s) for v, s in zip(vs, sg)])
    return Formula(n, clauses)


def record(name, n, ratio, fseed, threads, lw, gw, timeout, max_rounds):
    inserted = []
    results = []
    orig_insert = E.ClauseStore.insert
    orig_round = E.Engine.run_round
    orig_cfg = O.EngineConfig

    def insert(self, lits, engine_id, origin, activity):
        inserted.append((engine_id, tuple(lits)))
        return orig_insert(self, lits, engine_id, origin, activity)

    def run_round(self):
        r = orig_round(self)
        results.append((len(inserted), r))
        return r

    def traced_cfg(**kw):
        return orig_cfg(trace=True, **kw)

    engines = []
    orig_engine = O.Engine

    def make_engine(*a, **kw):
        e = orig_engine(*a, **kw)
        engines.append(e)
        return e

    E.ClauseStore.insert = insert
    E.Engine.run_round = run_round
    O.EngineConfig = traced_cfg
    O.Engine = make_engine
    try:
        ans = O.solve_parallel(random_3cnf(n, ratio, fseed),
                               O.RunConfig(threads=threads, lane_width=lw, group_width=gw, seed=fseed,
                                           timeout=timeout))
    finally:
        E.ClauseStore.insert = orig_insert
        E.Engine.run_round = orig_round
        O.EngineConfig = orig_cfg
        O.Engine = orig_engine
    eng = engines[0]
    assert [e for e, _ in inserted] == list(range(len(inserted))), "ids inserted out of order (drops?)"
    assert len(eng.trace) == len(results)
    out = {"num_vars": np.int64(n), "threads": np.int64(threads), "lane_width": np.int64(lw),
           "group_width": np.int64(gw), "status": np.array(ans.status.value)}
    lens = np.array([len(l) for _, l in inserted], np.int64)
    out["ins_off"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out["ins_lits"] = np.array([x for _, l in inserted for x in l], np.int32)
    k = 0
    for (n_ins, res), tr in zip(results, eng.trace):
        if not tr.snapshots:
            continue
        p = f"r{k}_"
        out[p + "n_inserted"] = np.int64(n_ins)
        out[p + "live"] = np.array(sorted(eid for eid, _ in tr.store), np.int64)
        out[p + "snap_tid"] = np.array([t for t, _ in tr.snapshots], np.int32)
        out[p + "snap_vals"] = np.stack([np.asarray(v, np.int8) for _, v in tr.snapshots])
        out[p + "rep_dest"] = np.array([r.destination for r in tr.reports], np.int32)
        out[p + "rep_eid"] = np.array([r.engine_id for r in tr.reports], np.int64)
        out[p + "rep_mask"] = np.array([r.lane_mask for r in tr.reports], np.uint64)
        out[p + "result"] = np.array([res.reports_emitted, res.clauses_tested, res.assignments_consumed,
                                      res.aggregate_tests_negative], np.int64)
        k += 1
        if k >= max_rounds:
            break
    out["rounds"] = np.int64(k)
    path = os.path.join(HERE, f"c5_replay_{name}.npz")
    np.savez_compressed(path, **out)
    chunks = max((len(np.unique(out[f"r{i}_snap_tid"])) for i in range(k)), default=0)
    print(f"{name}: {ans.status.value}, {k} rounds, {len(inserted)} clauses inserted, "
          f"{sum(len(out[f'r{i}_rep_eid']) for i in range(k))} reports, <= {chunks} threads per round "
          f"-> {path} ({os.path.getsize(path) // 1024} KB)")


if __name__ == "__main__":
    for name, args in CASES.items():
        record(name, *args)
