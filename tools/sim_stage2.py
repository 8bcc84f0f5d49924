"""Host-side model of k_test's stage 2 on the C3 generator: positive
(clause, group) pairs and warp iterations per tile by clause size -- where
stage 2's work is (profiles/r02_gather_ceiling.md).

    python tools/sim_stage2.py
"""
import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_03119_b200 import workload as W
cfg = W.CONFIGS['C3']; n = 200000
rng = np.random.default_rng(cfg.seed)
snaps = W.snapshots(cfg.threads, cfg.lanes, cfg.num_vars, np.random.default_rng(cfg.seed + 999))
V=cfg.num_vars; G=cfg.threads; L=cfg.lanes
s3 = snaps.reshape(G, L, V + 1)
cbT=(s3==1).any(1).T; cbF=(s3==-1).any(1).T; cbU=(s3==0).any(1).T
buckets = W.clause_buckets(n, V, rng)
iters=0; pairs=0; tiles=0; by_size={}
for s, arr in buckets.items():
    c=arr.shape[0]; var=np.abs(arr); neg=arr<0
    litF=np.where(neg[...,None], cbT[var], cbF[var]); litU=cbU[var]
    af=np.ones((c,G),bool); ou=np.zeros((c,G),bool)
    for j in range(s):
        ou=(af&litU[:,j])|(ou&litF[:,j]); af=af&litF[:,j]
    pos=(af|ou).sum(1)
    for t0 in range(0,c,32):
        p=pos[t0:t0+32]; it=p.max(); iters+=it; pairs+=p.sum(); tiles+=1
        d=by_size.setdefault(s,[0,0,0]); d[0]+=it; d[1]+=p.sum(); d[2]+=1
print("stage-2 iterations per tile", iters/tiles, "positive pairs per tile", pairs/tiles, "lane efficiency", pairs/(iters*32))
for s in sorted(by_size)[:8]:
    it,pp,t=by_size[s]; print(f"  size {s}: iters/tile {it/t:.1f} pairs/tile {pp/t:.1f} eff {pp/max(it*32,1):.2f}")
print("share of all iterations in sizes<=5:", sum(by_size[s][0] for s in by_size if s<=5)/iters)
