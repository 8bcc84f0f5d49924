"""Host-side model of k_test's stage-1 round trips per warp tile on the C3
generator: how many round trips a 32-clause tile needs (the warp runs until
its last live lane's recurrence ends) and how many lanes are live in each
(profiles/r02_gather_ceiling.md).

    python tools/sim_ragged.py
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
rt_total=0; lane_batches=0; gathers=0; tiles=0
rt_hist={}
for s, arr in buckets.items():
    c=arr.shape[0]; var=np.abs(arr); neg=arr<0
    litF=np.where(neg[...,None], cbT[var], cbF[var]); litU=cbU[var]
    af=np.ones((c,G),bool); ou=np.zeros((c,G),bool); la=[]
    for j in range(s):
        ou=(af&litU[:,j])|(ou&litF[:,j]); af=af&litF[:,j]; la.append((af|ou).any(1))
    la=np.stack(la,1)  # alive after literal j
    # schedule: batch [0,4), then [4,6), [6,8), then 4 at a time
    bounds=[0,4,6,8]+list(range(12, 200, 4))
    for t0 in range(0, c, 32):
        tl = la[t0:t0+32]; tiles+=1
        alive = np.ones(tl.shape[0], bool); rts=0
        for bi in range(len(bounds)-1):
            h0, h1 = bounds[bi], min(bounds[bi+1], s)
            if h0 >= s: break
            act = alive.sum()
            if act == 0: break
            rts += 1; lane_batches += act; gathers += act*(h1-h0)
            alive = alive & tl[:, h1-1]
        rt_total += rts; rt_hist[rts]=rt_hist.get(rts,0)+1
print("tiles", tiles, "mean warp round trips per tile (stage 1)", rt_total/tiles)
print("mean live lanes per round trip", lane_batches/rt_total)
print("histogram of round trips per tile:", dict(sorted(rt_hist.items())))
