"""The multi-GPU round (paper_2012_03119_b200/sharded.py ShardedRound) with
the real engine on every rank: world_size 2 sharing the one GPU of the test
box, gloo carrying the CUDA table broadcast and the record gather (the
deployment uses NCCL over NVLink, one rank per GPU; the data path is the
same calls).  Rank 0 stages and encodes, the tables are broadcast, every
rank tests its shard on the GPU, the records are merged in the reference
order -- and must equal the unsharded oracle's ordered report list."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NV, N, SEED = 3000, 40_000, 11


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    from paper_2012_03119_b200 import workload as W
    rng = np.random.default_rng(SEED)
    buckets = W.clause_buckets(N, NV, rng, 1, 12)
    flat, offs, ids = W.flatten(buckets)
    snaps = W.snapshots(5, 32, NV, rng)
    gl, gt = W.groups_for(5, 32, 16)  # lane_width 16 -> 10 groups; group_width 4 -> 3 chunks
    return buckets, flat, offs, ids, snaps, gl, gt


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2012_03119_b200 import sharded as S
    from paper_2012_03119_b200.native import NativeEngine

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        buckets, flat, offs, ids, snaps, gl, gt = _inputs()
        sizes = np.diff(offs)
        owner = S.assign_shards(sizes, world)
        mine = np.nonzero(owner == rank)[0]
        f = np.concatenate([flat[offs[i]:offs[i + 1]] for i in mine]) if len(mine) else np.zeros(0, np.int32)
        o = np.concatenate([[0], np.cumsum(sizes[mine])]).astype(np.int64)
        eng = NativeEngine(NV, 16, 4, device=0)
        eng.add_clauses(f, o, ids[mine])
        res, parts = S.ShardedRound(dist, eng, 4).run(gl, gt, 1.0, snaps if rank == 0 else None)
        if rank == 0:
            size_of = {int(ids[i]): int(sizes[i]) for i in range(len(ids))}
            brank = {s: k for k, s in enumerate(buckets.keys())}
            merged = S.merge_reports(parts, 4, brank, size_of)
            out_q.put(("ok", merged.tobytes()))
        eng.close()
    except Exception:
        import traceback
        out_q.put(("err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_sharded_round_on_gpu_matches_unsharded_oracle():
    from gpu_util import require_device
    require_device()
    from oracle import oracle as O
    from paper_2012_03119_b200.reports import DECODED_DTYPE

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, payload = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", payload
    merged = np.frombuffer(payload, dtype=DECODED_DTYPE)

    buckets, flat, offs, ids, snaps, gl, gt = _inputs()
    st = O.OracleStore()
    st.insert_flat(flat, offs, ids)
    want, _ = st.test_round(NV, snaps, gl, gt, 16, 4, 1.0)
    assert len(want) > 1000 and len(merged) == len(want)
    for fld in ("engine_id", "lane_mask", "group"):
        assert np.array_equal(merged[fld], want[fld]), fld


def _split_worker(rank, world, port, out_q):
    # split ingress: every rank stages + encodes only its
    # groups' rows; tables combined by all-gather + sum all-reduce
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2012_03119_b200 import sharded as S
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine, pack_rows

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(SEED + 1)
        buckets = W.clause_buckets(N, NV, rng, 1, 12)
        flat, offs, ids = W.flatten(buckets)
        snaps = W.snapshots(4, 32, NV, rng)
        gl, gt = W.groups_for(4, 32)
        sizes = np.diff(offs)
        owner = S.assign_shards(sizes, world)
        mine = np.nonzero(owner == rank)[0]
        f = np.concatenate([flat[offs[i]:offs[i + 1]] for i in mine])
        o = np.concatenate([[0], np.cumsum(sizes[mine])]).astype(np.int64)
        eng = NativeEngine(NV, 32, 32, device=0)
        eng.add_clauses(f, o, ids[mine])
        gb, ge = S.split_groups(len(gl), world, rank)
        rows = pack_rows(snaps[gb * 32:ge * 32], NV)
        res, parts = S.ShardedRound(dist, eng, 32).run_split(gl, gt, 1.0, rows)
        if rank == 0:
            size_of = {int(ids[i]): int(sizes[i]) for i in range(len(ids))}
            brank = {s: k for k, s in enumerate(buckets.keys())}
            merged = S.merge_reports(parts, 32, brank, size_of)
            out_q.put(("ok", merged.tobytes()))
        eng.close()
    except Exception:
        import traceback
        out_q.put(("err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_split_ingress_round_on_gpu_matches_unsharded_oracle():
    from gpu_util import require_device
    require_device()
    from oracle import oracle as O
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.reports import DECODED_DTYPE

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, payload = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", payload
    merged = np.frombuffer(payload, dtype=DECODED_DTYPE)

    rng = np.random.default_rng(SEED + 1)
    buckets = W.clause_buckets(N, NV, rng, 1, 12)
    flat, offs, ids = W.flatten(buckets)
    snaps = W.snapshots(4, 32, NV, rng)
    gl, gt = W.groups_for(4, 32)
    st = O.OracleStore()
    st.insert_flat(flat, offs, ids)
    want, _ = st.test_round(NV, snaps, gl, gt, 32, 32, 1.0)
    assert len(want) > 1000 and len(merged) == len(want)
    for fld in ("engine_id", "lane_mask", "group"):
        assert np.array_equal(merged[fld], want[fld]), fld
