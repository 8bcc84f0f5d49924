"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The fixtures were produced by running the reference (triggersat) itself; see
tests/golden/make_golden.py.  These tests need no GPU.
"""
import numpy as np
import pytest

from golden_io import bitpack_golden, engine_golden
from oracle import oracle as O

BP = bitpack_golden()


def test_pack_matches_reference():
    for case in BP["pack"]:
        t, s, m = O.pack(case["assignments"], case["num_vars"], case["lane_width"])
        assert [int(x) for x in t] == case["is_true"]
        assert [int(x) for x in s] == case["is_set"]
        assert m == case["lane_mask"]


def test_lane_trigger_matches_reference():
    for lane in BP["lane"]:
        case = BP["pack"][lane["case"]]
        t, s, m = O.pack(case["assignments"], case["num_vars"], case["lane_width"])
        got = [O.assignment_trigger(t, s, case["lane_width"], m, c) for c in lane["clauses"]]
        assert got == lane["masks"]


def test_aggregate_and_multi_trigger_match_reference():
    for case in BP["agg"]:
        nv, gw, lw = case["num_vars"], case["group_width"], case["lane_width"]
        packed = [O.pack(g, nv, lw) for g in case["groups"]]
        if not packed:
            assert all(w == 0 for w in case["words"])
            continue
        cbt, cbf, cbu = O.aggregate([(t, s) for t, s, _ in packed], [len(g) for g in case["groups"]], nv, gw)
        assert [int(x) for x in cbt] == case["can_be_true"]
        assert [int(x) for x in cbf] == case["can_be_false"]
        assert [int(x) for x in cbu] == case["can_be_undef"]
        for c, w, multi in zip(case["clauses"], case["words"], case["multi"]):
            word = O.aggregate_trigger(cbt, cbf, cbu, gw, len(packed), c)
            assert word == w
            got = []
            for i in range(len(packed)):
                if word >> i & 1:
                    t, s, m = packed[i]
                    mask = O.assignment_trigger(t, s, lw, m, c)
                    if mask:
                        got.append([i, mask])
            assert got == multi


def test_gate1_exhaustive_and_corpus():
    ex = BP["gate1_exhaustive"]
    t, s, m = O.pack(ex["assignments"], 3, 32)
    assert [O.assignment_trigger(t, s, 32, m, c) for c in ex["clauses"]] == ex["masks"]
    n = 0
    for case in BP["gate1_corpus"]:
        t, s, m = O.pack(case["assignments"], case["num_vars"], case["lane_width"])
        for c, want in zip(case["clauses"], case["masks"]):
            assert O.assignment_trigger(t, s, case["lane_width"], m, c) == want
            n += 1
    assert n == 20000


def _replay_oracle(spec, nthreads):
    eng = O.OracleEngine(spec["num_vars"], spec["threads"], nthreads=nthreads, **spec["config"])
    for op, exp in zip(spec["ops"], spec["expect"]):
        if op[0] == "add":
            assert eng.add_clause(op[1], op[2]) == exp["id"]
        elif op[0] == "submit":
            assert eng.submit_assignment(op[1], op[3], op[2]) == exp["ok"]
        else:
            if op[0] == "round":
                res = eng.run_round()
                assert [res["reports_emitted"], res["clauses_tested"], res["assignments_consumed"],
                        res["aggregate_tests_negative"]] == exp["result"]
            else:
                assert eng.reduce_store() == exp["removed"]
            for t in spec["observe_threads"]:
                got = [[list(r.lits), r.engine_id, r.lane_mask, r.destination] for r in eng.drain_reports(t)]
                assert got == exp["reports"][str(t)], (spec["name"], t)
            for k, v in eng.counters.items():
                assert exp["counters"][k] == v, (spec["name"], k)
            store = [[eid, list(l), o, float(a).hex()] for eid, l, o, a in eng.store.clauses()]
            assert store == exp["store"], spec["name"]
            assert float(eng.inc).hex() == exp["activity_inc"]


@pytest.mark.parametrize("nthreads", [1, 3])
def test_oracle_engine_replays_reference_scenarios(nthreads):
    for spec in engine_golden():
        _replay_oracle(spec, nthreads)
