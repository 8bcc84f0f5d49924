"""Synthetic workloads of SURVEY.md §8(d) (host-side numpy generators).

Clauses: size ~ U{2..30}, distinct variables uniform over 1..V, signs
Bernoulli(0.5).  Assignments: T solver threads x 32 lanes; per thread and
variable a value subset is drawn from the paper's window table
({T}.127 {F}.064 {U}.660 {T,U}.060 {F,U}.068 {T,F,U}.021)
and every lane draws uniformly inside the subset.  Slot 0 is Undef.

The generator is vectorised (per size bucket, duplicate-variable rows are
redrawn) so the 10M-clause config builds in seconds; it is seeded and
deterministic, but it is not the survey's per-clause rng stream.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Tuple

import numpy as np

SUBSET_P = np.array([0.127, 0.064, 0.660, 0.060, 0.068, 0.021])
SUBSET_P = SUBSET_P / SUBSET_P.sum()
# value choices per subset, padded to 3 entries; k = subset size
_SUB_VALS = np.array([[1, 1, 1], [-1, -1, -1], [0, 0, 0], [1, 0, 1], [-1, 0, -1], [1, -1, 0]], dtype=np.int8)
_SUB_K = np.array([1, 1, 1, 2, 2, 3])


@dataclass(frozen=True)
class Config:
    name: str
    n_clauses: int
    threads: int
    lanes: int
    num_vars: int
    size_lo: int = 2
    size_hi: int = 30
    seed: int = 20121

    @property
    def assignments(self) -> int:
        return self.threads * self.lanes


CONFIGS = {
    "C1": Config("C1", 100_000, 2, 32, 10_000, seed=20121 + 1),
    "C2": Config("C2", 1_000_000, 8, 32, 50_000, seed=20121 + 2),
    "C3": Config("C3", 10_000_000, 32, 32, 200_000, seed=20121 + 3),
}


def clause_buckets(n: int, num_vars: int, rng: np.random.Generator, size_lo=2, size_hi=30
                   ) -> Dict[int, np.ndarray]:
    """{size: int32[count, size]} with distinct variables per clause."""
    sizes = rng.integers(size_lo, size_hi + 1, n)
    counts = np.bincount(sizes, minlength=size_hi + 1)
    out = {}
    for s in range(size_lo, size_hi + 1):
        c = int(counts[s])
        if c == 0:
            continue
        if s == 0:
            out[s] = np.zeros((c, 0), np.int32)
            continue
        if s * s > num_vars // 4:  # dense: rejection would rarely succeed
            if s > num_vars:
                raise ValueError(f"clause size {s} exceeds {num_vars} variables")
            vs = np.stack([rng.choice(num_vars, s, replace=False) + 1 for _ in range(c)]).astype(np.int64)
            sign = rng.integers(0, 2, (c, s), dtype=np.int64) * 2 - 1
            out[s] = (vs * sign).astype(np.int32)
            continue
        vs = rng.integers(1, num_vars + 1, (c, s), dtype=np.int64)
        while True:
            srt = np.sort(vs, axis=1)
            bad = np.nonzero((srt[:, 1:] == srt[:, :-1]).any(axis=1))[0] if s > 1 else np.zeros(0, np.int64)
            if bad.size == 0:
                break
            vs[bad] = rng.integers(1, num_vars + 1, (bad.size, s), dtype=np.int64)
        sign = rng.integers(0, 2, (c, s), dtype=np.int64) * 2 - 1
        out[s] = (vs * sign).astype(np.int32)
    return out


def snapshots(threads: int, lanes: int, num_vars: int, rng: np.random.Generator) -> np.ndarray:
    """int8[threads*lanes, num_vars+1]; rows of thread t are t*lanes .. t*lanes+lanes-1."""
    out = np.empty((threads * lanes, num_vars + 1), dtype=np.int8)
    for t in range(threads):
        pick = rng.choice(6, num_vars + 1, p=SUBSET_P)
        k = _SUB_K[pick]
        u = (rng.random((lanes, num_vars + 1)) * k).astype(np.int64)
        rows = _SUB_VALS[pick[None, :], u]
        rows[:, 0] = 0
        out[t * lanes:(t + 1) * lanes] = rows
    return out


def flatten(buckets: Dict[int, np.ndarray], id0: int = 0) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(lits, offsets, ids) in bucket order, ready for tsg_add_clauses."""
    lits, offs, ids = [], [0], []
    nxt = id0
    total = 0
    for s, arr in buckets.items():
        lits.append(arr.reshape(-1))
        c = arr.shape[0]
        offs.append(total + s * np.arange(1, c + 1, dtype=np.int64))
        total += s * c
        ids.append(np.arange(nxt, nxt + c, dtype=np.int64))
        nxt += c
    flat = np.concatenate(lits).astype(np.int32) if lits else np.zeros(0, np.int32)
    off = np.concatenate([np.zeros(1, np.int64)] + offs[1:]) if len(offs) > 1 else np.zeros(1, np.int64)
    return flat, off, (np.concatenate(ids) if ids else np.zeros(0, np.int64))


def shard(buckets: Dict[int, np.ndarray], world: int, rank: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Rank `rank`'s clause shard of a store filled by `flatten(buckets)`:
    rows rank, rank + world, ... of every size bucket (balanced buckets,
    SURVEY.md §8(e)), with the global engine ids flatten assigns.  The union
    over ranks is the whole store."""
    sub: Dict[int, np.ndarray] = {}
    idl: List[np.ndarray] = []
    nxt = 0
    for s, arr in buckets.items():
        sub[s] = arr[rank::world]
        idl.append(nxt + np.arange(rank, arr.shape[0], world, dtype=np.int64))
        nxt += arr.shape[0]
    flat, off, _ = flatten(sub)
    return flat, off, (np.concatenate(idl) if idl else np.zeros(0, np.int64))


def in_reference_order(dec: np.ndarray, offsets: np.ndarray, ids: np.ndarray,
                       buckets: Dict[int, np.ndarray], group_width: int) -> np.ndarray:
    """Decoded report records (reports.decode) of a store filled by `flatten`
    (ids ascending from ids[0]), sorted in the reference emission order."""
    from .reports import reference_order
    sizes = np.diff(offsets)
    rank_of_size = np.zeros(max(buckets) + 1 if buckets else 1, np.int64)
    for k, s in enumerate(buckets):
        rank_of_size[s] = k
    brank = rank_of_size[sizes[dec["engine_id"] - ids[0]]] if len(dec) else np.zeros(0, np.int64)
    return dec[reference_order(dec, group_width, brank)]


def groups_for(threads: int, lanes: int, lane_width: int = 32) -> Tuple[np.ndarray, np.ndarray]:
    """Group lanes / tids of the reference grouping (engine.py:390-399) for
    `lanes` snapshots per thread, tids 0..threads-1."""
    gl: List[int] = []
    gt: List[int] = []
    for t in range(threads):
        for i in range(0, lanes, lane_width):
            gl.append(min(lane_width, lanes - i))
            gt.append(t)
    return np.asarray(gl, np.int32), np.asarray(gt, np.int32)
