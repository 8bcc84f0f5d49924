"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container only (it imports the reference from
/root/reference/pkg/src, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed, small):
  bitpack_golden.json   -- pack / aggregate / lane / aggregate-trigger / multi_trigger
                           known answers, incl. acceptance gate 1's exhaustive
                           27x26 block and a slice of its seed-20260825 corpus
  engine_golden.json    -- scripted Engine scenarios: per-round results, drained
                           reports in order, counters and exact store contents
                           (activities as float.hex) after every round

The fixture format is plain JSON so the CPU oracle tests and the GPU parity
tests can replay it without the reference.
"""
from __future__ import annotations

import itertools
import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")

from triggersat.bitpack import (  # noqa: E402
    aggregate_trigger,
    assignment_trigger,
    build_aggregate_batch,
    multi_trigger,
    pack_assignments,
)
from triggersat.core import FALSE, TRUE, UNDEF, all_undef  # noqa: E402
from triggersat.engine import AssignmentSnapshot, Engine, EngineConfig  # noqa: E402
from oracles import random_assignment, random_clause  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
VALUES = (TRUE, FALSE, UNDEF)


def rand_values(rng, nv, p_set=0.7):
    vals = [UNDEF] * (nv + 1)
    for v in range(1, nv + 1):
        if rng.random() < p_set:
            vals[v] = TRUE if rng.random() < 0.5 else FALSE
    return vals


def rand_clause(rng, nv, size):
    vs = rng.sample(range(1, nv + 1), size)
    return [v if rng.random() < 0.5 else -v for v in vs]


def bitpack_cases():
    rng = random.Random(20121)
    out = {"pack": [], "lane": [], "agg": [], "gate1_exhaustive": None, "gate1_corpus": []}
    # pack + lane trigger (bitpack.py:81-135), widths 1..64
    for _ in range(600):
        nv = rng.randint(1, 12)
        lw = rng.randint(1, 64)
        lanes = rng.randint(0, min(lw, 40))
        asg = [[UNDEF] + [rng.choice(VALUES) for _ in range(nv)] for _ in range(lanes)]
        b = pack_assignments(asg, nv, lw)
        clauses = [rand_clause(rng, nv, rng.randint(0, min(8, nv))) for _ in range(6)]
        out["pack"].append({
            "num_vars": nv, "lane_width": lw, "assignments": asg,
            "is_true": [int(x) for x in b.is_true], "is_set": [int(x) for x in b.is_set],
            "lane_mask": b.lane_mask,
        })
        out["lane"].append({
            "case": len(out["pack"]) - 1, "clauses": clauses,
            "masks": [assignment_trigger(b, c) for c in clauses],
        })
    # aggregate + aggregate_trigger + multi_trigger (bitpack.py:152-300)
    for _ in range(400):
        nv = rng.randint(1, 10)
        gw = rng.randint(1, 64)
        gc = rng.randint(0, min(gw, 12))
        lw = rng.choice([4, 8, 32, 64])
        groups = []
        for _ in range(gc):
            lanes = rng.randint(0, min(lw, 6))
            groups.append([[UNDEF] + [rng.choice(VALUES) for _ in range(nv)] for _ in range(lanes)])
        batches = [pack_assignments(g, nv, lw) for g in groups]
        agg = build_aggregate_batch(batches, gw)
        clauses = [rand_clause(rng, nv, rng.randint(0, min(6, nv))) for _ in range(6)]
        words, multis = [], []
        for c in clauses:
            words.append(aggregate_trigger(agg, c))
            got = []
            if batches:
                multi_trigger(agg, batches, c, lambda i, m: got.append([i, m]))
            multis.append(got)
        out["agg"].append({
            "num_vars": nv, "group_width": gw, "lane_width": lw, "groups": groups,
            "can_be_true": [int(x) for x in agg.can_be_true] if gc else [],
            "can_be_false": [int(x) for x in agg.can_be_false] if gc else [],
            "can_be_undef": [int(x) for x in agg.can_be_undef] if gc else [],
            "group_mask": agg.group_mask, "clauses": clauses, "words": words,
            "multi": multis,
        })
    # acceptance gate 1, exhaustive block (test_acceptance.py:101-118)
    asg = []
    for combo in itertools.product((TRUE, FALSE, UNDEF), repeat=3):
        v = all_undef(3)
        v[1:] = combo
        asg.append(v)
    b = pack_assignments(asg, 3, 32)
    clauses = []
    for size in (1, 2, 3):
        for vs in itertools.combinations((1, 2, 3), size):
            for signs in itertools.product((1, -1), repeat=size):
                clauses.append([s * v for s, v in zip(signs, vs)])
    out["gate1_exhaustive"] = {"assignments": asg, "clauses": clauses,
                               "masks": [assignment_trigger(b, c) for c in clauses]}
    # acceptance gate 1 corpus, first 400 batches (seed 20260825, test_acceptance.py:81-98)
    crng = random.Random(20260825)
    for _ in range(400):
        nv = crng.randint(1, 12)
        lanes = crng.randint(1, 32)
        lw = crng.randint(lanes, 32)
        lane_values = [random_assignment(crng, nv) for _ in range(lanes)]
        b = pack_assignments(lane_values, nv, lw)
        cls = []
        for _ in range(50):
            size = crng.randint(1, min(8, nv))
            cls.append(list(random_clause(crng, nv, size)))
        out["gate1_corpus"].append({"num_vars": nv, "lane_width": lw, "assignments": lane_values,
                                    "clauses": cls, "masks": [assignment_trigger(b, c) for c in cls]})
    return out


# ---------------------------------------------------------------------------
# engine scenarios

def observe(engine, threads, result):
    reports = {}
    for t in threads:
        reports[str(t)] = [[list(r.lits), r.engine_id, r.lane_mask, r.destination]
                           for r in engine.drain_reports(t)]
    counters = {k: v for k, v in engine.raw_counters().items() if k != "busy_seconds"}
    store = [[eid, list(lits), origin, float(act).hex()] for eid, lits, origin, act in engine.store.clauses()]
    buckets = [[size, int(b.count)] for size, b in engine.store.buckets.items()]
    return {
        "result": [result.reports_emitted, result.clauses_tested,
                   result.assignments_consumed, result.aggregate_tests_negative] if result else None,
        "reports": reports, "counters": counters, "store": store, "bucket_order": buckets,
        "activity_inc": float(engine._activity_inc).hex(),
    }


def run_scenario(spec):
    cfg = EngineConfig(**spec["config"])
    engine = Engine(spec["num_vars"], spec["threads"], cfg)
    obs = []
    for op in spec["ops"]:
        kind = op[0]
        if kind == "add":
            eid = engine.add_clause(tuple(op[1]), origin=op[2])
            obs.append({"op": "add", "id": eid})
        elif kind == "submit":
            vals = np.array(op[3], dtype=np.int8)
            ok = engine.submit_assignment(AssignmentSnapshot(op[1], vals, op[2]))
            obs.append({"op": "submit", "ok": ok})
        elif kind == "round":
            res = engine.run_round()
            o = observe(engine, spec["observe_threads"], res)
            o["op"] = "round"
            obs.append(o)
        elif kind == "reduce":
            n = engine.reduce_store()
            o = observe(engine, spec["observe_threads"], None)
            o["op"] = "reduce"
            o["removed"] = n
            obs.append(o)
    spec = dict(spec)
    spec["expect"] = obs
    return spec


def snap_vals(nv, mapping):
    v = [0] * (nv + 1)
    for k, w in mapping.items():
        v[k] = w
    return v


def scripted():
    S = []
    # test_engine.py:99-113
    S.append({"name": "route_fifo", "num_vars": 3, "threads": 2, "config": {}, "observe_threads": [0, 1],
              "ops": [["add", [1, 2], 0], ["add", [3], 0],
                      ["submit", 1, 0, snap_vals(3, {1: -1, 2: -1, 3: -1})],
                      ["submit", 0, 0, snap_vals(3, {1: 1, 3: 1})], ["round"], ["round"]]})
    # test_engine.py:119-132
    S.append({"name": "only_triggering", "num_vars": 5, "threads": 1, "config": {}, "observe_threads": [0],
              "ops": [["add", [1, 2], 0], ["add", [-3, 4], 0], ["add", [3, 5], 0], ["add", [4, 5], 0],
                      ["submit", 0, 0, snap_vals(5, {1: -1, 2: -1, 3: 1})], ["round"]]})
    # test_engine.py:135-145
    S.append({"name": "one_report_per_thread", "num_vars": 2, "threads": 1,
              "config": {"lane_width": 2, "assignment_queue_capacity": 8}, "observe_threads": [0],
              "ops": [["add", [1, 2], 0]] + [["submit", 0, i, snap_vals(2, {1: -1, 2: -1})] for i in range(5)]
              + [["round"]]})
    # test_engine.py:158-175
    S.append({"name": "counters", "num_vars": 3, "threads": 2, "config": {}, "observe_threads": [0, 1],
              "ops": [["add", [1, 2], 0], ["add", [-3], 1], ["submit", 0, 0, snap_vals(3, {1: 1})],
                      ["submit", 1, 0, snap_vals(3, {3: 1})], ["submit", 1, 1, snap_vals(3, {3: -1})], ["round"]]})
    # test_engine.py:205-216
    S.append({"name": "reduce_watermark", "num_vars": 4, "threads": 1, "config": {"reduce_keep_fraction": 0.5},
              "observe_threads": [0],
              "ops": [["add", [1, i + 2], 0] for i in range(4)] + [["round"], ["reduce"], ["reduce"]]})
    # test_engine.py:219-225
    S.append({"name": "capacity_drop", "num_vars": 4, "threads": 1, "config": {"max_clauses": 2},
              "observe_threads": [0], "ops": [["add", [1, i + 2], 0] for i in range(3)] + [["round"]]})
    # queue drop-newest, test_engine.py:88-96
    S.append({"name": "queue_drop", "num_vars": 2, "threads": 1, "config": {"assignment_queue_capacity": 2},
              "observe_threads": [0],
              "ops": [["submit", 0, 0, snap_vals(2, {1: 1})], ["submit", 0, 1, snap_vals(2, {1: -1})],
                      ["submit", 0, 2, snap_vals(2, {2: 1})], ["round"]]})
    # empty clause and unit clause on pad lanes (test_bitpack.py:93-98 at engine level)
    S.append({"name": "empty_and_unit", "num_vars": 1, "threads": 1, "config": {}, "observe_threads": [0],
              "ops": [["add", [], 0], ["add", [1], 0]] + [["submit", 0, i, [0, 0]] for i in range(3)] + [["round"]]})
    return S


def rand_clause_repeats(rng, nv, size):
    """Variables drawn with replacement: repeated literals and x / -x pairs."""
    return [rng.randint(1, nv) * (1 if rng.random() < 0.5 else -1) for _ in range(size)]


def randomized(seed, n_rounds, nv, threads, cfg, adds_per_round, snaps_per_round, p_set, size_hi,
               reduce_every=0, name=None, repeats=False):
    rng = random.Random(seed)
    ops = []
    seq = {t: 0 for t in range(threads)}
    for r in range(n_rounds):
        for _ in range(rng.randint(*adds_per_round)):
            size = rng.randint(0, min(size_hi, nv) if not repeats else size_hi)
            clause = rand_clause_repeats(rng, nv, size) if repeats else rand_clause(rng, nv, size)
            ops.append(["add", clause, rng.randrange(threads)])
        for _ in range(rng.randint(*snaps_per_round)):
            t = rng.randrange(threads)
            ops.append(["submit", t, seq[t], rand_values(rng, nv, p_set)])
            seq[t] += 1
        ops.append(["round"])
        if reduce_every and r % reduce_every == reduce_every - 1:
            ops.append(["reduce"])
    return {"name": name or f"random_{seed}", "num_vars": nv, "threads": threads, "config": cfg,
            "observe_threads": list(range(threads)), "ops": ops}


def engine_scenarios():
    S = scripted()
    # multi-chunk rounds with threads spanning chunk boundaries (engine.py:390-407)
    S.append(randomized(1, 6, 8, 3, {"lane_width": 2, "group_width": 3, "assignment_queue_capacity": 9},
                        (3, 12), (2, 14), 0.8, 4))
    S.append(randomized(2, 6, 10, 4, {"lane_width": 3, "group_width": 2, "assignment_queue_capacity": 7},
                        (5, 20), (4, 20), 0.7, 5))
    # capacity pressure -> reduce inside integrate, explicit reduces, ties on activity
    S.append(randomized(3, 8, 9, 2, {"max_clauses": 12, "lane_width": 4, "group_width": 2,
                                     "reduce_keep_fraction": 0.5},
                        (2, 9), (1, 8), 0.8, 4, reduce_every=3))
    S.append(randomized(4, 8, 12, 3, {"max_clauses": 30, "reduce_keep_fraction": 0.3, "lane_width": 64,
                                      "group_width": 64, "assignment_queue_capacity": 70},
                        (4, 15), (2, 70), 0.6, 6, reduce_every=2))
    # activity rescale (engine.py:416-420): inc grows 1e20 per round
    S.append(randomized(5, 9, 6, 2, {"activity_decay": 1e-20, "lane_width": 8, "group_width": 4},
                        (2, 6), (1, 10), 0.9, 3))
    # default widths, wide clauses
    S.append(randomized(6, 4, 40, 3, {}, (20, 60), (10, 40), 0.95, 30))
    S.append(randomized(7, 5, 16, 5, {"lane_width": 1, "group_width": 1, "assignment_queue_capacity": 3},
                        (3, 10), (2, 12), 0.85, 3))
    # repeated literals and tautologies (x or -x): the engine takes any literal list
    S.append(randomized(8, 6, 5, 2, {"lane_width": 8, "group_width": 4, "max_clauses": 40},
                        (4, 12), (2, 16), 0.7, 6, reduce_every=3, name="repeats_and_tautologies",
                        repeats=True))
    return [run_scenario(s) for s in S]


def main():
    with open(os.path.join(HERE, "bitpack_golden.json"), "w") as fh:
        json.dump(bitpack_cases(), fh, separators=(",", ":"))
    with open(os.path.join(HERE, "engine_golden.json"), "w") as fh:
        json.dump(engine_scenarios(), fh, separators=(",", ":"))
    for f in ("bitpack_golden.json", "engine_golden.json"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
