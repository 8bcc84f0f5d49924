"""SURVEY.md §8(f)3 / PAPER.md:425: the chunk-level ("32x32x32") aggregate,
measured on real CDCL snapshots and on the synthetic window-table ones.

1. Runs the reference's CDCL threads (baseline/_ref) with the GPU Engine on
   the C5 instance (random 3-SAT, n = 20000, ratio 4.26) for `secs` seconds,
   capturing every submitted snapshot and, at the end, the store of learned
   clauses.
2. Builds rounds of 32 chunks x 32 groups x 32 lanes (32768 assignments):
   each thread's snapshots in submission order, 32 per group, threads
   contiguous (engine.py:390-399 grouping).
3. Times the trigger kernel on two stores -- the learned clauses (replicated
   to `store` clauses) and random clauses of sizes U[2,30] -- with the
   chunk-level sweep on and off (TSG_CHUNK_FILTER), and reports the share of
   (clause, chunk) pairs it left for stage 1 (TSG_F_CHUNK_FILTER).  Records
   must be identical.

    python tools/hier_probe.py [secs=40] [store=4000000] > gpurun_out/hier_probe.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2012_03119_b200 import exchange as X  # noqa: E402
from paper_2012_03119_b200 import workload as W  # noqa: E402
from paper_2012_03119_b200.native import NativeEngine, pack_rows  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 40.0
n_store = int(sys.argv[2]) if len(sys.argv) > 2 else 4_000_000
NV, THREADS, CHUNKS = 20_000, 8, 32


def capture_solver(secs):
    import paper_2012_03119_b200.engine as E
    snaps = []
    orig = E.Engine.submit_assignment

    def sub(self, s):
        if len(snaps) < 60_000:
            snaps.append((s.thread_id, np.array(s.values, dtype=np.int8)))
        return orig(self, s)

    E.Engine.submit_assignment = sub
    engines = []
    try:
        formula = X.random_3cnf(NV, 4.26, 7)
        ans = X.run(formula, threads=THREADS, timeout=secs, seed=7, gpu=True, keep=engines)
        learned = [lits for _, lits, _, _ in engines[0].store.clauses()]
        status = ans.status.value
    finally:
        E.Engine.submit_assignment = orig
        for e in engines:
            e.close()
    return snaps, learned, status


def round_rows(snaps, per_thread_groups):
    """Rows for one round: every thread's first per_thread_groups * 32 snapshots."""
    by = {}
    for t, v in snaps:
        by.setdefault(t, []).append(v)
    rows, gl, gt = [], [], []
    for t in sorted(by):
        s = by[t][:per_thread_groups * 32]
        for i in range(0, len(s), 32):
            rows.extend(s[i:i + 32])
            gl.append(len(s[i:i + 32]))
            gt.append(t)
    return np.stack(rows), np.asarray(gl, np.int32), np.asarray(gt, np.int32)


def measure(flat, offs, ids, rows, gl, gt, reps=5):
    out = {}
    for filt in (1, 0):
        e = NativeEngine(NV, 32, 32, timing=True, report_capacity=1 << 22, chunk_filter=bool(filt))
        e.add_clauses(flat, offs, ids)
        e.stage_packed(pack_rows(rows, NV, threads=8))
        e.prepare(gl, gt)
        ms = []
        for _ in range(reps):
            e.encode()
            r = e.test(1.0)
            ms.append(r.test_ms)
        recs = np.sort(e.fetch(r.reports), order=["engine_id", "group"])
        out[filt] = dict(test_ms=float(np.median(ms[1:])), encode_ms=r.encode_ms, chunks=r.n_chunks,
                         clauses_tested=r.clauses_tested, chunk_positives=r.chunk_positives,
                         aggregate_tests_negative=r.aggregate_tests_negative, aggregate_tests=r.aggregate_tests,
                         reports=r.reports, recs=recs)
        e.close()
    same = np.array_equal(out[1].pop("recs"), out[0].pop("recs"))
    on, off = out[1], out[0]
    return {"test_ms_chunk_filter": on["test_ms"], "test_ms_no_filter": off["test_ms"],
            "speedup": off["test_ms"] / on["test_ms"], "chunks": on["chunks"],
            "chunk_pairs_left": on["chunk_positives"] / on["clauses_tested"],
            "negative_aggregate_ratio": on["aggregate_tests_negative"] / on["aggregate_tests"],
            "reports": on["reports"], "records_identical": bool(same),
            "encode_ms_32_chunks": on["encode_ms"]}


def main():
    if X.import_reference() is None:
        print(json.dumps({"unavailable": "reference package (baseline/_ref) not installed"}))
        return
    t0 = time.time()
    snaps, learned, status = capture_solver(secs)
    per = min(len([1 for t, _ in snaps if t == k]) for k in range(THREADS)) // 32
    per = min(per, CHUNKS * 32 // THREADS)
    rows, gl, gt = round_rows(snaps, per)
    rng = np.random.default_rng(11)
    syn = W.snapshots(THREADS, per * 32, NV, rng)
    res = {"instance": f"random 3-SAT n={NV} ratio 4.26 seed 7, {THREADS} reference CDCL threads, {secs:.0f} s "
                       f"({status}), GPU engine", "snapshots_captured": len(snaps),
           "round": f"{len(gl)} groups of 32 ({(len(gl) + 31) // 32} chunks of 32 groups), {rows.shape[0]} assignments",
           "learned_clauses": len(learned),
           "learned_mean_size": float(np.mean([len(c) for c in learned])) if learned else None}
    # store 1: the learned clauses, replicated to n_store
    if learned:
        lens = np.array([len(c) for c in learned], np.int64)
        base_flat = np.concatenate([np.asarray(c, np.int32) for c in learned])
        reps = max(1, n_store // len(learned))
        flat = np.tile(base_flat, reps)
        offs = np.concatenate([[0], np.cumsum(np.tile(lens, reps))]).astype(np.int64)
        ids = np.arange(len(lens) * reps, dtype=np.int64)
        res["learned_store"] = {"clauses": int(len(ids)),
                                "solver_snapshots": measure(flat, offs, ids, rows, gl, gt),
                                "synthetic_snapshots": measure(flat, offs, ids, syn, gl, gt)}
        del flat
    # store 2: random clauses of sizes U[2,30] (the SURVEY §8(d) generator)
    b = W.clause_buckets(n_store, NV, np.random.default_rng(12))
    flat, offs, ids = W.flatten(b)
    res["random_store"] = {"clauses": int(len(ids)),
                           "solver_snapshots": measure(flat, offs, ids, rows, gl, gt),
                           "synthetic_snapshots": measure(flat, offs, ids, syn, gl, gt)}
    res["wall_s"] = time.time() - t0
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
