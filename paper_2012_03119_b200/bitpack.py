"""Bit-parallel assignment batches and trigger tests, computed on the GPU.

Mirror of the reference's library API (bitpack.py:1-300): same names, same
argument meaning, same errors.  Every compute function runs the sm_100a
kernels of libtsg.so (tsg_pack / tsg_aggregate / tsg_lane_trigger /
tsg_aggregate_trigger); the dataclasses hold the resulting words as numpy
uint64 arrays in the reference layout (one word per variable, slot 0 unused)
so callers can inspect them exactly as before.  The batched variants
(`assignment_trigger_many`, `aggregate_trigger_many`) test many clauses in
one launch.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Iterator, List, Sequence

import numpy as np

from . import _lib
from ._lib import CapacityError, check, ptr

WORD_BITS = 64
_U64_ONE = np.uint64(1)

# value conventions of the reference (core.py:20-22): a variable is True,
# False or Undef; a literal is +v / -v; assignments are indexed by variable
# with slot 0 unused
TRUE, FALSE, UNDEF = 1, -1, 0

#: CUDA device used by the library-level kernels.
DEVICE = 0


def set_device(device: int) -> None:
    global DEVICE
    DEVICE = int(device)


def _check_width(width: int, what: str) -> None:  # bitpack.py:33-36
    if not 1 <= width <= WORD_BITS:
        raise ValueError(f"{what} must be in 1..{WORD_BITS}, got {width}")


def _flatten(clauses):
    offs = np.zeros(len(clauses) + 1, dtype=np.int64)
    for i, c in enumerate(clauses):
        offs[i + 1] = offs[i] + len(c)
    lits = np.zeros(max(int(offs[-1]), 1), dtype=np.int32)
    k = 0
    for c in clauses:
        n = len(c)
        if n:
            lits[k:k + n] = np.asarray(c, dtype=np.int32)
        k += n
    return lits, offs


@dataclass(frozen=True)
class PackedAssignmentBatch:
    """Up to ``lane_width`` assignments packed as per-variable bit words
    (bitpack.py:39-78)."""

    num_vars: int
    lane_width: int
    lane_count: int
    lane_mask: int
    is_true: np.ndarray
    is_set: np.ndarray

    def literal_words(self, lit: int) -> tuple:
        """(lanes where the literal's variable is set, lanes where the literal
        is False): a set lane is False for +v where v is not True, for -v
        where it is."""
        t, s = int(self.is_true[abs(lit)]), int(self.is_set[abs(lit)])
        false_lanes = s & (t if lit < 0 else ~t)
        return s, false_lanes

    def lane_assignment(self, lane: int) -> list:
        if not 0 <= lane < self.lane_count:
            raise IndexError(f"lane {lane} out of range (count {self.lane_count})")
        bit = _U64_ONE << np.uint64(lane)
        t = (self.is_true & bit) != 0
        s = (self.is_set & bit) != 0
        values = np.where(s, np.where(t, TRUE, FALSE), UNDEF)
        values[0] = UNDEF
        return [int(x) for x in values]


def pack_assignments(assignments: Sequence[Sequence[int]], num_vars: int,
                     lane_width: int = 32) -> PackedAssignmentBatch:
    """bitpack.py:81-117, encoded on the GPU (K1)."""
    _check_width(lane_width, "lane_width")
    if len(assignments) > lane_width:
        raise CapacityError(f"{len(assignments)} assignments exceed lane width {lane_width}")
    n = len(assignments)
    rows = np.zeros((max(n, 1), num_vars + 1), dtype=np.int8)
    for i, values in enumerate(assignments):
        vals = np.asarray(values, dtype=np.int8)
        if vals.shape[0] != num_vars + 1:
            raise ValueError(f"assignment {i} has {vals.shape[0]} slots, expected {num_vars + 1}")
        rows[i] = vals
    is_true = np.zeros(num_vars + 1, dtype=np.uint64)
    is_set = np.zeros(num_vars + 1, dtype=np.uint64)
    check(_lib.load().tsg_pack(DEVICE, ptr(rows), n, num_vars + 1, num_vars, lane_width,
                               ptr(is_true), ptr(is_set)))
    return PackedAssignmentBatch(num_vars=num_vars, lane_width=lane_width, lane_count=n,
                                 lane_mask=(1 << n) - 1, is_true=is_true, is_set=is_set)


def assignment_trigger_many(batch: PackedAssignmentBatch, clauses: Sequence[Sequence[int]]) -> List[int]:
    """Lane masks of many clauses against one batch, one kernel launch."""
    if not clauses:
        return []
    lits, offs = _flatten(clauses)
    out = np.zeros(len(clauses), dtype=np.uint64)
    check(_lib.load().tsg_lane_trigger(DEVICE, ptr(batch.is_true), ptr(batch.is_set), batch.num_vars,
                                       batch.lane_width, batch.lane_mask, ptr(lits), ptr(offs),
                                       len(clauses), ptr(out)))
    return [int(x) for x in out]


def assignment_trigger(batch: PackedAssignmentBatch, clause: Sequence[int]) -> int:
    """bitpack.py:120-135: bitmask of the lanes on which the clause triggers."""
    return assignment_trigger_many(batch, [tuple(clause)])[0]


@dataclass(frozen=True)
class AggregateAssignment:
    """Per-variable subset of the values a group takes (bitpack.py:138-182)."""

    num_vars: int
    has_true: np.ndarray
    has_false: np.ndarray
    has_undef: np.ndarray

    @classmethod
    def from_packed(cls, batch: PackedAssignmentBatch) -> "AggregateAssignment":
        agg = build_aggregate_batch([batch], 1)
        return cls(batch.num_vars, agg.can_be_true != 0, agg.can_be_false != 0, agg.can_be_undef != 0)

    def values_at(self, v: int) -> frozenset:
        """The values variable v takes somewhere in the group."""
        return frozenset(val for val, has in ((TRUE, self.has_true), (FALSE, self.has_false),
                                              (UNDEF, self.has_undef)) if has[v])


@dataclass(frozen=True)
class AggregateBatch:
    """Up to ``group_width`` aggregates packed per variable (bitpack.py:185-208)."""

    num_vars: int
    group_width: int
    group_count: int
    group_mask: int
    can_be_true: np.ndarray
    can_be_false: np.ndarray
    can_be_undef: np.ndarray

    def group_aggregate(self, i: int) -> AggregateAssignment:
        if not 0 <= i < self.group_count:
            raise IndexError(f"group {i} out of range (count {self.group_count})")
        bit = _U64_ONE << np.uint64(i)
        return AggregateAssignment(self.num_vars, (self.can_be_true & bit) != 0,
                                   (self.can_be_false & bit) != 0, (self.can_be_undef & bit) != 0)


def build_aggregate_batch(batches: Sequence[PackedAssignmentBatch], group_width: int = 32) -> AggregateBatch:
    """bitpack.py:211-244, aggregated on the GPU (K2)."""
    _check_width(group_width, "group_width")
    if len(batches) > group_width:
        raise CapacityError(f"{len(batches)} groups exceed group width {group_width}")
    if not batches:
        z = np.zeros(1, dtype=np.uint64)
        return AggregateBatch(0, group_width, 0, 0, z, z.copy(), z.copy())
    num_vars = batches[0].num_vars
    for b in batches:
        if b.num_vars != num_vars:
            raise ValueError("all batches must cover the same variable range")
    T = np.stack([b.is_true for b in batches]).astype(np.uint64)
    S = np.stack([b.is_set for b in batches]).astype(np.uint64)
    lanes = np.asarray([b.lane_count for b in batches], dtype=np.int32)
    out = np.zeros((3, num_vars + 1), dtype=np.uint64)
    check(_lib.load().tsg_aggregate(DEVICE, ptr(T), ptr(S), ptr(lanes), len(batches), num_vars, group_width,
                                    ptr(out[0]), ptr(out[1]), ptr(out[2])))
    return AggregateBatch(num_vars=num_vars, group_width=group_width, group_count=len(batches),
                          group_mask=(1 << len(batches)) - 1, can_be_true=out[0].copy(),
                          can_be_false=out[1].copy(), can_be_undef=out[2].copy())


def aggregate_trigger_many(agg: AggregateBatch, clauses: Sequence[Sequence[int]]) -> List[int]:
    """Aggregate words of many clauses, one kernel launch."""
    if not clauses:
        return []
    if agg.group_count == 0:
        return [0] * len(clauses)
    lits, offs = _flatten(clauses)
    out = np.zeros(len(clauses), dtype=np.uint64)
    check(_lib.load().tsg_aggregate_trigger(DEVICE, ptr(agg.can_be_true), ptr(agg.can_be_false),
                                            ptr(agg.can_be_undef), agg.num_vars, agg.group_width,
                                            agg.group_count, ptr(lits), ptr(offs), len(clauses), ptr(out)))
    return [int(x) for x in out]


def aggregate_trigger(agg: AggregateBatch, clause: Sequence[int]) -> int:
    """bitpack.py:247-271: bitmask of groups whose aggregate the clause triggers on."""
    return aggregate_trigger_many(agg, [tuple(clause)])[0]


def iter_set_bits(word: int) -> Iterator[int]:
    """Indices of the set bits of a word, ascending (bitpack.py:274-279)."""
    return (i for i in range(int(word).bit_length()) if (word >> i) & 1)


def multi_trigger(agg: AggregateBatch, per_group_batches: Sequence[PackedAssignmentBatch],
                  clause: Sequence[int], report: Callable[[int, int], None]) -> None:
    """bitpack.py:282-300: two-stage test; report(group, lane_mask) for exactly
    the groups with a genuinely triggering lane."""
    groups = list(iter_set_bits(aggregate_trigger(agg, clause)))  # stage 1 on the GPU
    masks = [assignment_trigger(per_group_batches[i], clause) for i in groups]  # stage 2 per positive group
    for i, mask in zip(groups, masks):
        if mask:  # a positive aggregate without a triggering lane is not reported
            report(i, mask)
