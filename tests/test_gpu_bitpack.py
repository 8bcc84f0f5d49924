"""Library-level kernels (bitpack API) on the GPU vs the reference's own
outputs (golden fixtures) and vs the CPU oracle.  Mirrors the reference's
tests/test_bitpack.py and acceptance gates 1-3."""
import random

import numpy as np
import pytest

from golden_io import bitpack_golden
from gpu_util import require_device
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    require_device()
    import paper_2012_03119_b200 as P
    return P


@pytest.fixture(scope="module")
def BP():
    return bitpack_golden()


def test_pack_and_lane_trigger_match_reference(P, BP):
    for case, lane in zip(BP["pack"], BP["lane"]):
        b = P.pack_assignments(case["assignments"], case["num_vars"], case["lane_width"])
        assert [int(x) for x in b.is_true] == case["is_true"]
        assert [int(x) for x in b.is_set] == case["is_set"]
        assert b.lane_mask == case["lane_mask"]
        assert P.assignment_trigger_many(b, lane["clauses"]) == lane["masks"]
        for i, a in enumerate(case["assignments"]):
            assert b.lane_assignment(i) == list(a)


def test_aggregate_and_multi_trigger_match_reference(P, BP):
    for case in BP["agg"]:
        nv, gw, lw = case["num_vars"], case["group_width"], case["lane_width"]
        batches = [P.pack_assignments(g, nv, lw) for g in case["groups"]]
        agg = P.build_aggregate_batch(batches, gw)
        if batches:
            assert [int(x) for x in agg.can_be_true] == case["can_be_true"]
            assert [int(x) for x in agg.can_be_false] == case["can_be_false"]
            assert [int(x) for x in agg.can_be_undef] == case["can_be_undef"]
        assert agg.group_mask == case["group_mask"]
        assert P.aggregate_trigger_many(agg, case["clauses"]) == case["words"]
        for c, multi in zip(case["clauses"], case["multi"]):
            got = []
            if batches:
                P.multi_trigger(agg, batches, c, lambda i, m: got.append([i, m]))
            assert got == multi


def test_gate1_exhaustive_and_corpus(P, BP):
    ex = BP["gate1_exhaustive"]
    b = P.pack_assignments(ex["assignments"], 3, 32)
    assert P.assignment_trigger_many(b, ex["clauses"]) == ex["masks"]
    for case in BP["gate1_corpus"]:
        b = P.pack_assignments(case["assignments"], case["num_vars"], case["lane_width"])
        assert P.assignment_trigger_many(b, case["clauses"]) == case["masks"]


def test_known_answers(P):
    # test_bitpack.py:93-98 pad lanes stay silent; empty clause triggers on valid lanes
    b = P.pack_assignments([[0, 0]] * 3, 1, lane_width=32)
    assert P.assignment_trigger(b, (1,)) == 0b111
    assert P.assignment_trigger(b, ()) == 0b111
    # test_bitpack.py:187-199 aggregate false positive filtered by the lane test
    batch = P.pack_assignments([[0, 1, -1], [0, -1, 1]], 2, 8)
    agg = P.build_aggregate_batch([batch], 8)
    assert P.aggregate_trigger(agg, (1, 2)) == 1
    assert P.assignment_trigger(batch, (1, 2)) == 0
    got = []
    P.multi_trigger(agg, [batch], (1, 2), lambda i, m: got.append((i, m)))
    assert got == []
    # test_bitpack.py:248-252 empty group aggregates to all-Undef
    e = P.AggregateAssignment.from_packed(P.pack_assignments([], 2, 8))
    assert e.values_at(1) == frozenset({0}) and e.values_at(2) == frozenset({0})
    assert list(P.iter_set_bits(0b1011)) == [0, 1, 3]


def test_errors(P):
    # test_bitpack.py:101-112, 234-245
    with pytest.raises(P.CapacityError):
        P.pack_assignments([[0, 0]] * 3, 1, lane_width=2)
    with pytest.raises(ValueError):
        P.pack_assignments([], 1, lane_width=0)
    with pytest.raises(ValueError):
        P.pack_assignments([], 1, lane_width=65)
    with pytest.raises(ValueError):
        P.pack_assignments([[0]], 2, lane_width=4)
    with pytest.raises(IndexError):
        P.pack_assignments([[0, 1]], 1, 8).lane_assignment(1)
    b1, b2 = P.pack_assignments([], 3, 8), P.pack_assignments([], 4, 8)
    with pytest.raises(ValueError):
        P.build_aggregate_batch([b1, b2], 8)
    with pytest.raises(P.CapacityError):
        P.build_aggregate_batch([b1, b1, b1], 2)
    with pytest.raises(IndexError):
        P.build_aggregate_batch([b1], 8).group_aggregate(1)


def test_random_widths_vs_oracle(P):
    rng = random.Random(5)
    for _ in range(60):
        nv = rng.randint(1, 40)
        lw = rng.randint(1, 64)
        lanes = rng.randint(0, lw)
        asg = [[0] + [rng.choice((1, -1, 0)) for _ in range(nv)] for _ in range(lanes)]
        clauses = [[v if rng.random() < .5 else -v for v in rng.sample(range(1, nv + 1), rng.randint(0, min(nv, 12)))]
                   for _ in range(40)]
        b = P.pack_assignments(asg, nv, lw)
        t, s, m = O.pack(asg, nv, lw)
        assert np.array_equal(b.is_true, t) and np.array_equal(b.is_set, s)
        assert P.assignment_trigger_many(b, clauses) == [O.assignment_trigger(t, s, lw, m, c) for c in clauses]
