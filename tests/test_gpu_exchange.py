"""C5: the reference's CDCL solver threads exchanging
clauses through the GPU Engine (paper_2012_03119_b200/exchange.py), with the
reference orchestrator unchanged.

* The answer agrees with the reference engine's run on the same instance
  (both are complete solvers; SAT models are verified by the orchestrator).
* Every traced round's reports are sound and complete against the CPU oracle
  for that round's store and snapshots (acceptance gate 6 of the reference,
  test_acceptance.py:382-442), so solver threads import exactly the clauses
  the reference engine would have reported.

The live-loop tests need the reference package (baseline/_ref); the
replay test below does not: it feeds the GPU Engine the reference solver's
recorded rounds (tests/golden/c5_replay_*.npz, tests/golden/make_c5_replay.py)
and checks every drained report list against what the reference engine
delivered.
"""
import numpy as np
import pytest

from gpu_util import require_device
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def X():
    require_device()
    from paper_2012_03119_b200 import exchange as X
    if X.import_reference() is None:
        pytest.skip("reference package not installed (baseline/_ref)")
    return X


@pytest.mark.parametrize("name,devices,chunk_filter,ring", [("w32", None, False, 0), ("w8x2", None, False, 0),
                                                            ("w8x2", None, True, 0), ("w8x2", [0, 0], True, 0),
                                                            ("w32", None, False, 1024), ("w8x2", [0, 0], False, 128)])
def test_replay_reference_solver_rounds(name, devices, chunk_filter, ring):
    # every recorded round rebuilt on the GPU Engine through the reference API:
    # the same clauses under the same engine ids (inserted in id order, so the
    # size buckets are created in the reference's order), the round's
    # snapshots submitted per thread, then run_round and drain_reports --
    # per-destination report lists (engine id, lane mask, literals) in the
    # reference's order and the RoundResult must be identical
    require_device()
    import paper_2012_03119_b200 as P
    from golden_io import c5_replays, c5_round
    fx = c5_replays()[name]
    nv, th, lw, gw = (int(fx[k]) for k in ("num_vars", "threads", "lane_width", "group_width"))
    n_reports = 0
    for k in range(int(fx["rounds"])):
        clauses, live, snaps, reps, result = c5_round(fx, k)
        eng = P.Engine(nv, th, P.EngineConfig(lane_width=lw, group_width=gw, devices=devices,
                                              chunk_filter=chunk_filter, report_ring=ring))
        for lits in clauses:
            eng.add_clause(lits, origin=0)
        eng.run_round()  # integrate (no snapshots: no activity or counter effects)
        eng.remove_clauses([e for e in range(len(clauses)) if e not in live])
        for i, (tid, v) in enumerate(snaps):
            assert eng.submit_assignment(P.AssignmentSnapshot(int(tid), v, i))
        r = eng.run_round()
        assert [r.reports_emitted, r.clauses_tested, r.assignments_consumed, r.aggregate_tests_negative] == result
        for t in range(th):
            got = [(d.engine_id, d.lane_mask, d.lits) for d in eng.drain_reports(t)]
            want = [(e, m, clauses[e]) for dst, e, m in reps if dst == t]
            assert got == want, (name, k, t)
        n_reports += len(reps)
        eng.close()
    assert n_reports > 0


def check_trace(eng, nv):
    lw, gw = eng.config.lane_width, eng.config.group_width
    checked = 0
    for tr in eng.trace:
        if not tr.snapshots:
            continue
        by_tid = {}
        for tid, values in tr.snapshots:
            by_tid.setdefault(tid, []).append(values)
        rows, lanes, tids = [], [], []
        for tid in sorted(by_tid):
            s = by_tid[tid]
            for i in range(0, len(s), lw):
                rows.extend(s[i:i + lw])
                lanes.append(len(s[i:i + lw]))
                tids.append(tid)
        st = O.OracleStore()
        for eid, lits in tr.store:
            st.insert(list(lits), eid, 0, 1.0)
        recs, _ = st.test_round(nv, np.stack(rows), lanes, tids, lw, gw, 1.0)
        lits_of = dict(tr.store)
        want = sorted((tids[int(r["group"])], int(r["engine_id"]), int(r["lane_mask"]),
                       tuple(lits_of[int(r["engine_id"])])) for r in recs)
        got = sorted((r.destination, r.engine_id, r.lane_mask, tuple(r.lits)) for r in tr.reports)
        assert got == want
        checked += 1
    return checked


@pytest.mark.parametrize("seed", [0, 1, 3])  # n=150 near threshold: SAT, UNSAT, SAT
def test_exchange_loop_matches_reference_engine(X, seed):
    formula = X.random_3cnf(150, 4.26, seed)
    ref = X.run(formula, threads=4, timeout=120, seed=seed, gpu=False)
    engines = []
    ans = X.run(formula, threads=4, timeout=120, seed=seed, gpu=True, trace=True, keep=engines)
    assert ans.status.value != "UNKNOWN" and ans.status == ref.status
    s = X.summary(ans)
    assert s["engine_rounds"] > 0
    check_trace(engines[0], formula.num_vars)  # every round that tested snapshots
    for e in engines:
        e.close()


def test_exchange_loop_reports_are_imported(X):
    # a harder instance: long enough to exchange clauses, then verify that
    # the solver threads drained and imported what the GPU reported
    formula = X.random_3cnf(150, 4.26, 2)  # UNSAT, ~100 exchange rounds
    engines = []
    ans = X.run(formula, threads=4, timeout=120, seed=2, gpu=True, trace=True, keep=engines)
    assert ans.status.value == "UNSATISFIABLE"
    s = X.summary(ans)
    assert s["snapshots_submitted"] > 0 and s["clauses_exported"] > 0
    assert s["reports_drained"] <= ans.engine_counters["reports_delivered"]
    assert check_trace(engines[0], formula.num_vars) > 0
    for e in engines:
        e.close()


def test_reference_cli_with_gpu_engine(X, tmp_path):
    # the reference's CLI end to end (DIMACS, answer line, exit code,
    # --stats-json schema of instrumentation.py) with the GPU engine inside
    import io
    import json
    import contextlib
    from paper_2012_03119_b200.__main__ import main
    f = X.random_3cnf(150, 4.26, 1)  # UNSAT (checked against the reference engine above)
    cnf = tmp_path / "f.cnf"
    cnf.write_text(f"p cnf {f.num_vars} {len(f.clauses)}\n" +
                   "".join(" ".join(map(str, c)) + " 0\n" for c in f.clauses))
    stats = tmp_path / "stats.jsonl"
    out = io.StringIO()
    with contextlib.redirect_stdout(out):
        rc = main([str(cnf), "--threads", "4", "--timeout", "120", "--stats-json", str(stats)])
    assert rc == 20 and "s UNSATISFIABLE" in out.getvalue()
    rows = [json.loads(line) for line in stats.read_text().splitlines() if line.strip()]
    keys = set().union(*rows)
    assert any("imports_per_assignment" in str(r) for r in rows), keys
