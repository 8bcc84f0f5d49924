"""Host-side timing of each C-ABI call in the pipelined e2e loop (diagnostics)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2012_03119_b200 import _lib, workload as W  # noqa: E402
from paper_2012_03119_b200.native import NativeEngine, pack_rows, packed_words  # noqa: E402

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
rng = np.random.default_rng(cfg.seed)
b = W.clause_buckets(cfg.n_clauses, cfg.num_vars, rng)
flat, offs, ids = W.flatten(b)
eng = NativeEngine(cfg.num_vars, report_capacity=8 << 20)
eng.add_clauses(flat, offs, ids)
snaps = W.snapshots(cfg.threads, cfg.lanes, cfg.num_vars, np.random.default_rng(cfg.seed + 999))
gl, gt = W.groups_for(cfg.threads, cfg.lanes)
A = snaps.shape[0]
pw = packed_words(cfg.num_vars)
hp = torch.empty((A, pw), dtype=torch.int64).pin_memory()
pack_rows(snaps, cfg.num_vars, out=hp.numpy().view(np.uint64), threads=8)
bufs = [torch.empty((8 << 20) * 16, dtype=torch.uint8).pin_memory() for _ in range(2)]
L = eng.L
T = {}


def t(name, fn):
    t0 = time.perf_counter()
    r = fn()
    T.setdefault(name, []).append((time.perf_counter() - t0) * 1e3)
    return r


eng.set_record_bytes(8)
eng.prepare(gl, gt)
pending = 0
w0 = time.perf_counter()
for i in range(24):
    t("stage", lambda: _lib.check(L.tsg_stage_packed(eng.h, C.c_void_p(hp.data_ptr()), A, pw, 0)))
    if pending:
        r = t("collect", lambda: eng.collect())
        got = C.c_int64(0)
        t("fetch_async", lambda: _lib.check(L.tsg_fetch_reports_async(
            eng.h, C.c_void_p(bufs[i % 2].data_ptr()), r.reports, C.byref(got))))
        pending -= 1
    t("encode", lambda: eng.encode())
    t("launch", lambda: eng.launch(1.0))
    pending += 1
    if i == 3:
        w0 = time.perf_counter()
t("collect", lambda: eng.collect())
t("wait", lambda: eng.wait())
print(f"steady ms/step {(time.perf_counter() - w0) / 20 * 1e3:.3f}")
for k, v in T.items():
    print(f"{k:12s} median {np.median(v):8.3f} ms  max {max(v):8.3f}")
