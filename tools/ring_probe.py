"""Report egress through the host ring vs the device record buffer.

Per config, rounds from pinned 2-bit rows, synchronous (stage -> round ->
all records on the host), in two egress modes:

  buffer  records in HBM, then tsg_fetch_reports_async into pinned memory + wait
  ring_N  records written by k_test into the mapped host ring, drained by N
          CPU threads (RingDrainer) while the kernel runs

Reports the median wall ms per round (until the host holds every record),
the trigger kernel's event time in each mode and the record count; then
the same comparison through the drop-in Engine.run_round (EngineConfig
report_ring) for the configs other than C3.

    python tools/ring_probe.py [C1,C2,C3] [rounds=20] > gpurun_out/ring_probe.json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_03119_b200 import _lib  # noqa: E402
from paper_2012_03119_b200 import workload as W  # noqa: E402
from paper_2012_03119_b200.native import NativeEngine, RingDrainer, pack_rows  # noqa: E402

names = (sys.argv[1] if len(sys.argv) > 1 else "C1,C2,C3").split(",")
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 20


def pinned_copy(a: np.ndarray) -> tuple:
    import ctypes as C
    p = C.c_void_p()
    _lib.check(_lib.load().tsg_host_alloc(a.nbytes, C.byref(p)))
    buf = np.ctypeslib.as_array((C.c_uint8 * a.nbytes).from_address(p.value)).view(a.dtype).reshape(a.shape)
    buf[...] = a
    return buf, p


def probe(name):
    cfg = W.CONFIGS[name]
    rng = np.random.default_rng(cfg.seed)
    b = W.clause_buckets(cfg.n_clauses, cfg.num_vars, rng)
    flat, offs, ids = W.flatten(b)
    eng = NativeEngine(cfg.num_vars, timing=True, report_capacity=8 << 20)
    eng.add_clauses(flat, offs, ids)
    del flat, b
    snaps = W.snapshots(cfg.threads, cfg.lanes, cfg.num_vars, np.random.default_rng(cfg.seed + 999))
    gl, gt = W.groups_for(cfg.threads, cfg.lanes)
    rows, rows_p = pinned_copy(pack_rows(snaps, cfg.num_vars, threads=os.cpu_count() or 8))
    out = {"config": name, "clauses": cfg.n_clauses, "assignments": int(snaps.shape[0])}
    # buffer mode
    recs, recs_p = pinned_copy(np.zeros(8 << 20, _lib.REPORT_DTYPE))
    wall, kern = [], []
    for r in range(rounds + 3):
        t0 = time.perf_counter()
        eng.stage_packed(rows)
        res = eng.round(gl, gt, 1.0)
        eng.fetch_async(recs[:res.reports])
        eng.wait()
        t1 = time.perf_counter()
        if r >= 3:
            wall.append((t1 - t0) * 1e3)
            kern.append(res.test_ms)
    n_rec = res.reports
    out["buffer"] = {"ms_per_round": float(np.median(wall)), "k_test_ms": float(np.median(kern))}
    # ring, drained after the round by the calling thread (the drain loop alone)
    eng.ring_open(capacity=1 << 23, wait_ms=10_000)
    wall, drain = [], []
    buf = np.zeros(n_rec + 1, _lib.REPORT_DTYPE)
    try:
        for r in range(rounds + 3):
            t0 = time.perf_counter()
            eng.stage_packed(rows)
            res = eng.round(gl, gt, 1.0)
            t1 = time.perf_counter()
            k = 0
            while k < n_rec:  # one contiguous run per call
                k += len(eng.ring_drain(n_rec - k, timeout_ms=1000, out=buf[k:]))
            t2 = time.perf_counter()
            assert k == n_rec
            if r >= 3:
                wall.append((t2 - t0) * 1e3)
                drain.append((t2 - t1) * 1e3)
    finally:
        eng.ring_close()
    out["ring_after"] = {"ms_per_round": float(np.median(wall)), "drain_ms": float(np.median(drain))}
    # ring mode, 1 / 4 / 8 drainer threads
    for nd in (1, 4, 8):
        eng.ring_open(capacity=1 << 22, wait_ms=10_000)
        dr = RingDrainer(eng, threads=nd, batch=1 << 15)
        wall, kern = [], []
        try:
            for r in range(rounds + 3):
                t0 = time.perf_counter()
                eng.stage_packed(rows)
                res = eng.round(gl, gt, 1.0)
                got = dr.take(res.reports)
                t1 = time.perf_counter()
                assert len(got) == res.reports == n_rec
                if r >= 3:
                    wall.append((t1 - t0) * 1e3)
                    kern.append(res.test_ms)
        finally:
            dr.close()
            eng.ring_close()
        out[f"ring_{nd}"] = {"ms_per_round": float(np.median(wall)), "k_test_ms": float(np.median(kern))}
    out["records_per_round"] = int(n_rec)
    eng.close()
    for p in (rows_p, recs_p):
        _lib.load().tsg_host_free(p)
    return out




def api_probe(name, rounds=30):
    """Engine.run_round (the drop-in API) with the device record buffer vs the
    report ring: median ms per round."""
    import paper_2012_03119_b200 as P
    cfg = W.CONFIGS[name]
    out = {"config": name, "api": True}
    for ring in (0, 1 << 16):
        rng = np.random.default_rng(cfg.seed)
        flat, offs, _ = W.flatten(W.clause_buckets(cfg.n_clauses, cfg.num_vars, rng))
        eng = P.Engine(cfg.num_vars, cfg.threads, P.EngineConfig(max_clauses=2 * cfg.n_clauses, report_ring=ring,
                                                                assignment_queue_capacity=cfg.lanes))
        eng.add_clauses(flat, offs)
        eng.run_round()
        snaps = W.snapshots(cfg.threads, cfg.lanes, cfg.num_vars, np.random.default_rng(cfg.seed + 999))
        ms, reps = [], 0
        for r in range(rounds + 3):
            for i in range(snaps.shape[0]):
                eng.submit_assignment(P.AssignmentSnapshot(i // cfg.lanes, snaps[i], i))
            t0 = time.perf_counter()
            res = eng.run_round()
            t1 = time.perf_counter()
            for t in range(cfg.threads):
                eng.drain_reports(t)
            if r >= 3:
                ms.append((t1 - t0) * 1e3)
            reps = res.reports_emitted
        out["ring" if ring else "buffer"] = {"run_round_ms": float(np.median(ms))}
        out["reports_per_round"] = reps
        eng.close()
    return out


if __name__ == "__main__":
    for n in names:
        print(json.dumps(probe(n)), flush=True)
    for n in names:
        if n != "C3":
            print(json.dumps(api_probe(n)), flush=True)
