"""Count the random-sector traffic of the trigger test on a sample of a config
(host-side model of k_test, used to decide where gathers can be cut).

    python tools/sim_gathers.py [C3] [n_clauses]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_03119_b200 import workload as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
cfg = W.CONFIGS[name]
rng = np.random.default_rng(cfg.seed)
snaps = W.snapshots(cfg.threads, cfg.lanes, cfg.num_vars, np.random.default_rng(cfg.seed + 999))
V = cfg.num_vars
G = cfg.threads
L = cfg.lanes
s3 = snaps.reshape(G, L, V + 1)
T = (s3 == 1)
F = (s3 == -1)
U = (s3 == 0)
cbT = T.any(1).T  # [V+1, G]
cbF = F.any(1).T
cbU = U.any(1).T
# lane words as bool [V+1, G, L]
isT = T.transpose(2, 0, 1)
isF = F.transpose(2, 0, 1)
isU = U.transpose(2, 0, 1)

buckets = W.clause_buckets(n, V, rng)
tot = dict(rows=0, s1=0, s2=0, s2_mixed=0, clauses=0, pos=0, s1_ideal=0)
for s, arr in buckets.items():
    c = arr.shape[0]
    var = np.abs(arr)
    neg = arr < 0
    # per literal per group: nonF (lit can't be False) and U
    litF = np.where(neg[..., None], cbT[var], cbF[var])  # [c, s, G]
    litU = cbU[var]
    af = np.ones((c, G), bool)
    ou = np.zeros((c, G), bool)
    live_after = []
    for j in range(s):
        ou = (af & litU[:, j]) | (ou & litF[:, j])
        af = af & litF[:, j]
        live_after.append((af | ou).any(1))
    live_after = np.stack(live_after, 1)  # [c, s]
    # kernel: first 4 always, then batches of 2 up to 8, then batches of 4
    g1 = np.full(c, min(s, 4))
    h = 4
    while h < min(s, 8):
        alive = live_after[:, h - 1]
        g1 += alive * min(2, s - h)
        h += 2
    h = 8
    while h < s:
        alive = live_after[:, h - 1]
        g1 += alive * min(4, s - h)
        h += 4
    # ideal one-at-a-time
    ideal = 1 + live_after[:, :-1].sum(1) if s > 0 else np.zeros(c)
    tot["s1"] += g1.sum()
    tot["s1_ideal"] += ideal.sum()
    # rows: min(s,8) rows * 4 sectors per tile of 32
    tiles = (c + 31) // 32
    tot["rows"] += tiles * min(s, 8) * 4
    pos = af | ou  # [c, G]
    tot["pos"] += pos.sum()
    # stage 2: per positive (clause, group) lane gathers: batches of 4 for first 8, then 1 at a time
    ci, gi = np.nonzero(pos)
    if len(ci):
        lits = arr[ci]
        vv = var[ci]
        ng = neg[ci]
        lt = isT[vv, gi[:, None]]  # [p, s, L]
        lf = isF[vv, gi[:, None]]
        lu = isU[vv, gi[:, None]]
        litFalse = np.where(ng[..., None], lt, lf)
        a = np.ones((len(ci), L), bool)
        o = np.zeros((len(ci), L), bool)
        la = []
        for j in range(s):
            o = (a & lu[:, j]) | (o & litFalse[:, j])
            a = a & litFalse[:, j]
            la.append((a | o).any(1))
        la = np.stack(la, 1)
        g2 = np.full(len(ci), min(s, 4))
        if s > 4:
            g2 += la[:, 3] * min(4, s - 4)
        for j in range(8, s):
            g2 += la[:, j - 1]
        tot["s2"] += g2.sum()
        # mixed-subset literals among gathered ones (lower bound proxy: all literals mixed fraction)
        sub_single = ~((lt.any(2) & lf.any(2)) | (lt.any(2) & lu.any(2)) | (lf.any(2) & lu.any(2)))
        tot["s2_mixed"] += (~sub_single).sum() / max(1, s) * g2.mean() * 0 + 0
    tot["clauses"] += c
N = tot["clauses"]
print(f"{name}: {N} clauses sampled")
for k in ("rows", "s1", "s1_ideal", "s2", "pos"):
    print(f"  {k:10s} {tot[k] / N:.3f} per clause")
print(f"  total sectors/clause (rows+s1+s2) = {(tot['rows'] + tot['s1'] + tot['s2']) / N:.3f}")
