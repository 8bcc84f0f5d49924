"""Host-side logic of the multi-GPU path, world_size 2 on gloo (CPU).

The product's shard assignment, record gather/merge and exact global
reduce (paper_2012_03119_b200/sharded.py: select_prefix / global_reduce,
histograms summed over the process group) are exercised across two real
processes; each rank's shard compute is done here by the CPU oracle and a
numpy stand-in for tsg_reduce_begin/hist/commit (test infrastructure), and
the merged result must equal the unsharded oracle run: same ordered report
list, same reduce victims."""
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


class OracleShard:
    """tsg_reduce_begin / hist / commit over an oracle store (numpy), the
    interface sharded.global_reduce drives."""

    def __init__(self, st):
        self.st = st

    def reduce_begin(self, eligible_below):
        b = self.st.buckets()
        acts = np.concatenate([x[5] for x in b]) if b else np.zeros(0)
        ids = np.concatenate([x[3] for x in b]) if b else np.zeros(0, np.int64)
        el = ids < eligible_below
        self.a = acts[el].view(np.uint64).astype(object)
        self.i = ids[el].astype(object)
        return int(el.sum())

    def _top(self, bits):
        key = [(int(a) << 64) | int(i) for a, i in zip(self.a, self.i)]
        return [k >> (128 - bits) if bits else 0 for k in key], key

    def reduce_hist(self, ph, pl, bits):
        pref = ((ph << 64) | pl) >> (128 - bits) if bits else 0
        top, key = self._top(bits)
        h = np.zeros(256, np.int64)
        for t, k in zip(top, key):
            if t == pref:
                h[(k >> (120 - bits)) & 0xFF] += 1
        return h

    def reduce_commit(self, ph, pl, bits):
        if bits == 0:
            return np.zeros(0, np.int64)
        pref = ((ph << 64) | pl) >> (128 - bits)
        top, key = self._top(bits)
        doomed = [int(k & ((1 << 64) - 1)) for t, k in zip(top, key) if t <= pref]
        self.st.remove(doomed)
        return np.sort(np.asarray(doomed, np.int64))


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2012_03119_b200 import sharded as S
    from paper_2012_03119_b200 import workload as W

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
        parts = S.gather_records(dist, R.decode(R.encode(recs["engine_id"], recs["group"], recs["lane_mask"])), 0)
        a_all = S.gather_records(dist, np.zeros(0, R.DECODED_DTYPE), 0)  # empty gather
        # exact global reduce: histograms summed over the ranks
        removed, victims = S.global_reduce([OracleShard(st)], 10 ** 9, 1500, S.allreduce_np(dist))
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


def test_select_prefix_is_exact():
    # the radix select over shards: exactly k keys <= the selected prefix,
    # with heavy activity ties (ids break them, engine.py:488-489)
    from paper_2012_03119_b200.sharded import select_prefix
    rng = np.random.default_rng(1)
    shards = []
    for n in (50, 70, 0):
        acts = rng.integers(0, 5, n).astype(np.float64).view(np.uint64).astype(object)
        ids = rng.permutation(10 ** 6)[:n].astype(object)
        shards.append([(int(a) << 64) | int(i) for a, i in zip(acts, ids)])
    keys = sorted(sum(shards, []))

    def hist(ph, pl, bits):
        pref = ((ph << 64) | pl) >> (128 - bits) if bits else 0
        h = np.zeros(256, np.int64)
        for k in keys:
            if (k >> (128 - bits) if bits else 0) == pref:
                h[(k >> (120 - bits)) & 0xFF] += 1
        return h

    for k in (1, 17, 60, 119, 120):
        ph, pl, bits = select_prefix(hist, k)
        pref = ((ph << 64) | pl) >> (128 - bits)
        assert sum(1 for x in keys if x >> (128 - bits) <= pref) == k
        assert max(x for x in keys if x >> (128 - bits) <= pref) == keys[k - 1]
    assert select_prefix(hist, 0) == (0, 0, 0)


def test_split_groups_equal_contiguous_shares():
    # split ingress (sharded.combine_tables) needs equal contiguous group
    # shares so the group-major lane entries all-gather in place
    from paper_2012_03119_b200 import sharded as S
    assert S.split_groups(32, 1, 0) is None
    assert S.split_groups(30, 4, 0) is None
    got = [S.split_groups(32, 8, r) for r in range(8)]
    assert got[0] == (0, 4) and got[7] == (28, 32)
    assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
