"""Host-side logic of the multi-GPU path, world_size 2 on gloo (CPU).

The product's shard assignment, record gather/merge and exact global-reduce
threshold (paper_2012_03119_b200/sharded.py) are exercised across two real
processes; each rank's shard compute is done here by the CPU oracle (test
infrastructure), and the merged result must equal the unsharded oracle run:
same ordered report list, same reduce victims."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2012_03119_b200 import sharded as S
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200._lib import REPORT_DTYPE

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        nv = 400
        rng = np.random.default_rng(5)
        buckets = W.clause_buckets(6000, nv, rng, 1, 10)
        flat, offs, ids = W.flatten(buckets)
        sizes = np.diff(offs)
        owner = S.assign_shards(sizes, world)
        # every rank sees the same assignment; keep own clauses in arrival order
        mine = np.nonzero(owner == rank)[0]
        st = O.OracleStore()
        for i in mine:
            st.insert(flat[offs[i]:offs[i + 1]].tolist(), int(ids[i]), 0, 1.0)
        snaps = S.bcast_array(dist, W.snapshots(3, 32, nv, rng) if rank == 0 else None, 0, np.int8)
        snaps = snaps.reshape(-1, nv + 1)
        gl, gt = W.groups_for(3, 32, 16)  # lane_width 16 -> 6 groups
        recs, ctr = st.test_round(nv, snaps, gl, gt, 16, 4, 1.0)  # group_width 4 -> 2 chunks
        from paper_2012_03119_b200 import reports as R
        parts = S.gather_records(dist, R.encode(recs["engine_id"], recs["group"], recs["lane_mask"]), 0)
        # global reduce: gather eligible keys, exact threshold, local victim counts
        acts = np.concatenate([b[5] for b in st.buckets()]) if st.buckets() else np.zeros(0)
        kid = np.concatenate([b[3] for b in st.buckets()]) if st.buckets() else np.zeros(0, np.int64)
        a_all = S.gather_records(dist, np.zeros(0, REPORT_DTYPE), 0)  # empty gather
        keyparts = [None] * world
        dist.all_gather_object(keyparts, (acts, kid))
        thr = S.kth_key(keyparts, 1500)
        local = S.count_le(acts, kid, thr)
        removed, victims = st.reduce(10 ** 9, local)
        all_victims = [None] * world
        dist.all_gather_object(all_victims, sorted(victims.tolist()))
        if rank == 0:
            size_of = {int(ids[i]): int(sizes[i]) for i in range(len(ids))}
            brank = {s: k for k, s in enumerate(buckets.keys())}
            merged = S.merge_reports(parts, 4, brank, size_of)
            out_q.put(("ok", merged.tobytes(), sorted(sum(all_victims, [])), a_all is not None))
    except Exception as e:  # surface failures to the parent
        import traceback
        out_q.put(("err", traceback.format_exc(), None, None))
    finally:
        dist.destroy_process_group()


def test_two_rank_round_and_reduce_match_unsharded_oracle():
    from oracle import oracle as O
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200._lib import REPORT_DTYPE

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, merged, victims, _ = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", merged
    from paper_2012_03119_b200.reports import DECODED_DTYPE
    merged = np.frombuffer(merged, dtype=DECODED_DTYPE)

    # unsharded oracle on the same inputs
    nv = 400
    rng = np.random.default_rng(5)
    buckets = W.clause_buckets(6000, nv, rng, 1, 10)
    flat, offs, ids = W.flatten(buckets)
    st = O.OracleStore()
    st.insert_flat(flat, offs, ids)
    snaps = W.snapshots(3, 32, nv, rng)
    gl, gt = W.groups_for(3, 32, 16)
    want, _ = st.test_round(nv, snaps, gl, gt, 16, 4, 1.0)
    assert len(want) > 0
    for f in ("engine_id", "lane_mask", "group"):
        assert np.array_equal(merged[f], want[f]), f
    n, vict = st.reduce(10 ** 9, 1500)
    assert sorted(vict.tolist()) == victims


def test_assign_shards_balances_every_bucket():
    from paper_2012_03119_b200.sharded import assign_shards
    sizes = np.random.default_rng(0).integers(2, 31, 10_000)
    owner = assign_shards(sizes, 4)
    for s in np.unique(sizes):
        c = np.bincount(owner[sizes == s], minlength=4)
        assert c.max() - c.min() <= 1


def test_kth_key_and_count_le_are_exact():
    from paper_2012_03119_b200.sharded import count_le, kth_key
    rng = np.random.default_rng(1)
    acts = [rng.integers(0, 5, 50).astype(float), rng.integers(0, 5, 70).astype(float)]
    ids = [rng.permutation(200)[:50].astype(np.int64), 200 + rng.permutation(200)[:70].astype(np.int64)]
    for k in (1, 17, 60, 120):
        thr = kth_key(list(zip(acts, ids)), k)
        assert sum(count_le(a, i, thr) for a, i in zip(acts, ids)) == k
    assert kth_key(list(zip(acts, ids)), 500) is None


def test_split_groups_equal_contiguous_shares():
    # split ingress (sharded.combine_tables) needs equal contiguous group
    # shares so the group-major lane entries all-gather in place
    from paper_2012_03119_b200 import sharded as S
    assert S.split_groups(32, 1, 0) is None
    assert S.split_groups(30, 4, 0) is None
    got = [S.split_groups(32, 8, r) for r in range(8)]
    assert got[0] == (0, 4) and got[7] == (28, 32)
    assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
