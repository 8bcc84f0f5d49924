"""Device step time of back-to-back C3 rounds (two in flight) with and
without the per-round timing events (diagnostics for the value leg)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2012_03119_b200 import workload as W  # noqa: E402
from paper_2012_03119_b200.native import NativeEngine, pack_rows, packed_words  # noqa: E402

cfg = W.CONFIGS["C3"]
rng = np.random.default_rng(cfg.seed)
flat, offs, ids = W.flatten(W.clause_buckets(cfg.n_clauses, cfg.num_vars, rng))
snaps = W.snapshots(cfg.threads, cfg.lanes, cfg.num_vars, np.random.default_rng(cfg.seed + 999))
gl, gt = W.groups_for(cfg.threads, cfg.lanes)
A = snaps.shape[0]
pw = packed_words(cfg.num_vars)
d_packed = torch.from_numpy(pack_rows(snaps, cfg.num_vars, threads=16).view(np.int64)).cuda()
for timing in (True, False, True, False):
    eng = NativeEngine(cfg.num_vars, timing=timing, report_capacity=8 << 20)
    eng.add_clauses(flat, offs, ids)
    eng.stage_packed_ptr(d_packed.data_ptr(), A, pw, on_device=True)
    eng.prepare(gl, gt)
    st = torch.cuda.ExternalStream(eng.stream())

    def run(n):
        for i in range(n):
            if i >= 2:
                eng.collect()
            eng.encode()
            eng.launch(1.0)
        for _ in range(min(n, 2)):
            eng.collect()

    run(5)
    eng.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    run(40)
    b.record(st)
    eng.sync()
    b.synchronize()
    print(f"timing={timing} ms/step {a.elapsed_time(b) / 40:.4f}")
    eng.close()
