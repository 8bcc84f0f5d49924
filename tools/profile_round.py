"""Run a few device-resident rounds of a config (for ncu / nsys-less profiling).

    python tools/profile_round.py [C3] [rounds]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2012_03119_b200 import workload as W  # noqa: E402
from paper_2012_03119_b200.native import NativeEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = W.CONFIGS[name]
n_clauses = int(os.environ.get("TSG_N_CLAUSES", cfg.n_clauses))  # scale the store (capacity runs)
rng = np.random.default_rng(cfg.seed)
b = W.clause_buckets(n_clauses, cfg.num_vars, rng)
flat, offs, ids = W.flatten(b)
eng = NativeEngine(cfg.num_vars, timing=True, report_capacity=8 << 20)
eng.set_record_bytes(int(os.environ.get("TSG_RECORD_BYTES", "8")))  # as bench.py: the kernel writes 8-byte records
eng.add_clauses(flat, offs, ids)
del flat, b
snaps = W.snapshots(cfg.threads, cfg.lanes, cfg.num_vars, np.random.default_rng(cfg.seed + 999))
gl, gt = W.groups_for(cfg.threads, cfg.lanes)
if os.environ.get("TSG_INT8_ROWS"):  # int8 snapshot rows
    pitch = (cfg.num_vars + 1 + 15) // 16 * 16
    d = torch.zeros((snaps.shape[0], pitch), dtype=torch.int8, device="cuda")
    d[:, :cfg.num_vars + 1] = torch.from_numpy(snaps).cuda()
    torch.cuda.synchronize()
    eng.stage_device(d.data_ptr(), snaps.shape[0], pitch)
else:  # packed rows (the ingress format)
    from paper_2012_03119_b200.native import pack_rows, packed_words
    d = torch.from_numpy(pack_rows(snaps, cfg.num_vars, threads=8).view(np.int64)).cuda()
    torch.cuda.synchronize()
    eng.stage_packed_ptr(d.data_ptr(), snaps.shape[0], packed_words(cfg.num_vars), on_device=True)
eng.prepare(gl, gt)
for r in range(rounds):
    eng.encode()
    res = eng.test(1.0)
    print(f"round {r}: clauses {n_clauses} encode {res.encode_ms:.3f} ms test {res.test_ms:.3f} ms "
          f"({res.lane_tests / (res.test_ms * 1e-3):.3e} tests/s) reports {res.reports} "
          f"lane_triggers {res.lane_triggers} neg {res.aggregate_tests_negative}/{res.aggregate_tests}", flush=True)
