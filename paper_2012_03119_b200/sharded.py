"""Multi-GPU sharding of the clause store.

Clauses are tested independently, so the store shards by
clause: every shard owns a disjoint set of clauses in its own HBM store.  One
round (engine.py:369-467) becomes

    shard 0: stage + encode the round's snapshots (K1/K2)
    all    : replicate the packed tables over NVLink     <- the only data-path collective
or, with the snapshot ingress split:
    shard r: stage + encode the rows of its 1/N of the groups only (its own PCIe link)
    all    : all-gather the lane entries + sum-all-reduce the aggregate words
then
    all    : test the local shard (K3/K4/K5)
    all    : gather the report records, merge in the reference order

Two drivers use it: the Engine itself when EngineConfig.devices names
several GPUs (one process, one engine per device, tables copied peer to
peer: tsg_round_tables_copy), and one process per GPU under
torch.distributed (NCCL; `ShardedRound`, bench.py).  The global
reduce_store (engine.py:469-505) is exact in both: the doomed set is "the
`target` smallest (activity, engine_id) keys among eligible clauses", found
by a radix select whose per-pass histograms are summed over the shards
(`select_prefix`, tsg_reduce_begin/hist/commit), after which every shard
removes exactly its keys <= the selected prefix.

The pure host logic (shard assignment, record merge, prefix selection) is
tested on CPU with world_size 2 over gloo (tests/test_sharded_gloo.py).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import reports


# ---------------------------------------------------------------------------
# pure host logic

def assign_shards(sizes: Sequence[int], world: int, load: Optional[Dict[Tuple[int, int], int]] = None
                  ) -> np.ndarray:
    """Rank of every incoming clause: the rank holding the fewest clauses of
    that size so far (ties -> lowest rank), so every size bucket -- and with
    it the literal bytes -- is balanced across shards.
    `load[(size, rank)]` is updated in place."""
    load = {} if load is None else load
    out = np.empty(len(sizes), dtype=np.int32)
    for i, s in enumerate(sizes):
        s = int(s)
        best, best_n = 0, None
        for r in range(world):
            n = load.get((s, r), 0)
            if best_n is None or n < best_n:
                best, best_n = r, n
        out[i] = best
        load[(s, best)] = best_n + 1
    return out


def merge_reports(parts: Sequence[np.ndarray], group_width: int, bucket_rank_of: Dict[int, int],
                  size_of_eid: Dict[int, int]) -> np.ndarray:
    """Merge per-shard records (raw egress records or decoded) into the
    reference's report order.

    Within a bucket, slot order equals engine-id order (clauses are appended
    in id order and compaction preserves order, engine.py:150-163,184-200),
    so (chunk, global bucket rank, engine_id, group) is the unsharded order
    (engine.py:403-464) no matter which shard holds a clause.  Returns decoded
    records (reports.DECODED_DTYPE)."""
    raw = [p if p.dtype == reports.DECODED_DTYPE else reports.decode(p) for p in parts if len(p)]
    dec = np.concatenate(raw) if raw else np.zeros(0, reports.DECODED_DTYPE)
    if len(dec) == 0:
        return dec
    brank = reports.bucket_ranks(dec, size_of_eid, bucket_rank_of)
    return dec[reports.reference_order(dec, group_width, brank)]


def select_prefix(hist, k: int) -> Tuple[int, int, int]:
    """Steer the radix select of the k smallest 128-bit keys (activity bits,
    engine id) over any number of shards: `hist(prefix_hi, prefix_lo, bits)`
    returns the 256-bin histogram of the next 8 key bits, summed over the
    shards, among keys whose top `bits` bits equal the prefix.  Returns the
    prefix and its length such that exactly k keys have top bits <= it
    (bits = 0 and nothing selected when k == 0)."""
    ph = pl = bits = 0
    while k > 0 and bits < 128:
        h = np.asarray(hist(ph, pl, bits), dtype=np.int64)
        d = 0
        while d < 256 and h[d] < k:
            k -= int(h[d])
            d += 1
        if d == 256:
            raise RuntimeError("reduce select: the histograms lost keys")
        if bits < 64:
            ph |= d << (56 - bits)
        else:
            pl |= d << (120 - bits)
        bits += 8
        if h[d] == k:
            break
    return ph, pl, bits


def global_reduce(engines, eligible_below: int, target: int, allreduce=None) -> Tuple[int, np.ndarray]:
    """reduce_store over clause shards (engine.py:469-505), exact: remove the
    `target` smallest (activity, engine_id) keys among clauses with id <
    eligible_below across all `engines` (NativeEngine shards of this
    process).  `allreduce(np.int64 array) -> summed array` extends the sum
    over other processes (torch.distributed).  Returns (removed count here,
    removed ids here, ascending)."""
    ar = allreduce or (lambda a: a)
    n_el = ar(np.array([sum(e.reduce_begin(eligible_below) for e in engines)], np.int64))[0]
    rem = int(min(target, n_el))

    def hist(ph, pl, bits):
        return ar(np.sum([e.reduce_hist(ph, pl, bits) for e in engines], axis=0).astype(np.int64))

    ph, pl, bits = select_prefix(hist, rem) if rem > 0 else (0, 0, 0)
    gone = [e.reduce_commit(ph, pl, bits) for e in engines]
    ids = np.sort(np.concatenate(gone)) if gone else np.zeros(0, np.int64)
    return len(ids), ids


# ---------------------------------------------------------------------------
# array collectives over torch.distributed (NCCL on GPUs, gloo on CPU)

def _device(dist):
    import torch
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def bcast_array(dist, arr: Optional[np.ndarray], src: int, dtype) -> np.ndarray:
    import torch
    dev = _device(dist)
    n = torch.tensor([0 if arr is None else arr.size], dtype=torch.int64, device=dev)
    dist.broadcast(n, src)
    buf = torch.empty(int(n.item()), dtype=getattr(torch, np.dtype(dtype).name), device=dev)
    if dist.get_rank() == src and buf.numel():
        buf.copy_(torch.from_numpy(np.ascontiguousarray(arr, dtype=dtype).reshape(-1)).to(dev))
    if buf.numel():
        dist.broadcast(buf, src)
    return buf.cpu().numpy()


def gather_records(dist, recs: np.ndarray, dst: int = 0) -> Optional[List[np.ndarray]]:
    """Gather variable-length decoded record arrays (reports.DECODED_DTYPE)
    to `dst` only: sizes first (all-gather of one int), then a gather of
    the padded byte views."""
    import torch
    dev = _device(dist)
    world = dist.get_world_size()
    raw = np.ascontiguousarray(recs, dtype=reports.DECODED_DTYPE).view(np.uint8)
    n = torch.tensor([raw.size], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(x.item()) for x in sizes]
    m = max(sizes)
    if m == 0:
        return [np.zeros(0, reports.DECODED_DTYPE) for _ in range(world)] if dist.get_rank() == dst else None
    buf = torch.zeros(m, dtype=torch.uint8, device=dev)
    if raw.size:
        buf[:raw.size] = torch.from_numpy(raw).to(dev)
    bufs = [torch.zeros(m, dtype=torch.uint8, device=dev) for _ in range(world)] if dist.get_rank() == dst else None
    dist.gather(buf, bufs, dst=dst)
    if dist.get_rank() != dst:
        return None
    return [b[:k].cpu().numpy().view(reports.DECODED_DTYPE) for b, k in zip(bufs, sizes)]


def allreduce_np(dist):
    """np.int64 array -> its sum over the process group (for global_reduce)."""
    import torch
    dev = _device(dist)

    def f(a):
        t = torch.from_numpy(np.ascontiguousarray(a, np.int64)).to(dev)
        dist.all_reduce(t)
        return t.cpu().numpy()
    return f


def broadcast_tables(dist, engine, src: int = 0, stream=None) -> None:
    """Broadcast the round's packed tables (tsg_round_tables) from `src` to
    every rank, in place, over NCCL (NVLink on one node)."""
    import torch
    ptr, nbytes = engine.tables()

    class _CAI:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3, "stream": None}

    t = torch.as_tensor(_CAI(), device=torch.device("cuda", torch.cuda.current_device()))
    if stream is not None:
        with torch.cuda.stream(stream):
            dist.broadcast(t, src)
    else:
        dist.broadcast(t, src)


def split_groups(n_groups: int, world: int, rank: int) -> Optional[Tuple[int, int]]:
    """This rank's contiguous group range when the snapshot ingress is split
    (equal shares, so the lane tables all-gather in place); None if the
    groups do not divide evenly."""
    if world <= 1 or n_groups % world:
        return None
    per = n_groups // world
    return rank * per, (rank + 1) * per


def combine_tables(dist, engine, n_groups: int, stream=None) -> None:
    """After every rank encoded its group range (tsg_round_encode_groups):
    all-gather the lane entries (group-major, equal contiguous shares) and
    sum-all-reduce the aggregate words (each rank set only its groups' bits,
    so the sum is their OR) -- SURVEY.md §8(e)'s split ingress, in place on
    the round's table slot."""
    import torch
    ptr, nbytes = engine.tables()
    agg_off, agg_len, lane_off, gbytes = engine.layout()
    world, rank = dist.get_world_size(), dist.get_rank()

    class _CAI:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3, "stream": None}

    t = torch.as_tensor(_CAI(), device=torch.device("cuda", torch.cuda.current_device()))
    per = n_groups // world * gbytes
    lane = t[lane_off:lane_off + world * per]
    agg = t[agg_off:agg_off + agg_len].view(torch.int32)
    ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream())
    with ctx:
        mine = lane[rank * per:(rank + 1) * per]
        if dist.get_backend() == "nccl":
            dist.all_gather_into_tensor(lane, mine.clone())
        else:
            parts = [lane[r * per:(r + 1) * per] for r in range(world)]
            dist.all_gather(parts, mine.clone())
        dist.all_reduce(agg, op=dist.ReduceOp.SUM)


# ---------------------------------------------------------------------------
# the sharded round over NativeEngine shards

class ShardedRound:
    """One rank's side of a sharded exchange round (used by bench.py and by
    the distributed engine front end)."""

    def __init__(self, dist, engine, group_width: int = 32):
        import torch
        self.dist, self.eng, self.gw = dist, engine, group_width
        self.rank = dist.get_rank()
        self.stream = torch.cuda.ExternalStream(engine.stream())

    def run_split(self, group_lanes, group_tid, activity_inc: float, packed_rows: np.ndarray):
        """Split ingress: every rank passes the packed rows of its own group
        range only (split_groups), encodes them, and the tables are combined
        over the collective before every rank tests its shard."""
        n_groups = len(group_lanes)
        gb, ge = split_groups(n_groups, self.dist.get_world_size(), self.rank)
        self.eng.prepare(group_lanes, group_tid)
        self.eng.stage_packed(packed_rows)
        self.eng.encode_groups(gb, ge, self.rank == 0)
        # the collectives run on the engine's own stream: ordered after the
        # encode and before the test without a host sync
        combine_tables(self.dist, self.eng, n_groups, self.stream)
        res = self.eng.test(activity_inc)
        return res, gather_records(self.dist, self.eng.fetch(res.reports), 0)

    def run(self, group_lanes, group_tid, activity_inc: float, rows: Optional[np.ndarray] = None):
        """Rank 0 passes the round's grouped rows; every rank passes the same
        group_lanes / group_tid (broadcast by the caller)."""
        self.eng.prepare(group_lanes, group_tid)
        if self.rank == 0:
            if rows is not None:
                self.eng.stage(rows)
            self.eng.encode()
        broadcast_tables(self.dist, self.eng, 0, self.stream)  # on the engine's stream, after the encode
        res = self.eng.test(activity_inc)
        return res, gather_records(self.dist, self.eng.fetch(res.reports), 0)

    def reduce(self, eligible_below: int, target: int) -> Tuple[int, np.ndarray]:
        """The exact global reduce_store over every rank's shard."""
        return global_reduce([self.eng], eligible_below, target, allreduce_np(self.dist))
