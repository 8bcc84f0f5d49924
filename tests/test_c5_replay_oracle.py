"""The CPU oracle on the reference solver's recorded exchange rounds
(tests/golden/c5_replay_*.npz, made by running the reference itself): every
round's reports, in the reference's emission order, and its figures.  Pins
the oracle on real CDCL snapshots (similar trails per thread), where the
synthetic generators draw independent ones."""
import numpy as np

from golden_io import c5_replays, c5_round
from oracle import oracle as O


def test_oracle_matches_reference_on_solver_rounds():
    fxs = c5_replays()
    assert set(fxs) >= {"w32", "w8x2"}
    for name, fx in fxs.items():
        nv, lw, gw = int(fx["num_vars"]), int(fx["lane_width"]), int(fx["group_width"])
        multi = 0
        for k in range(int(fx["rounds"])):
            clauses, live, snaps, reps, result = c5_round(fx, k)
            st = O.OracleStore()
            for eid, lits in enumerate(clauses):
                if eid in live:
                    st.insert(list(lits), eid, 0, 1.0)
            by_tid = {}
            for tid, v in snaps:
                by_tid.setdefault(tid, []).append(v)
            rows, gl, gt = [], [], []
            for tid in sorted(by_tid):
                s = by_tid[tid]
                for i in range(0, len(s), lw):
                    rows.extend(s[i:i + lw])
                    gl.append(len(s[i:i + lw]))
                    gt.append(tid)
            multi += len(gl) > gw
            recs, ctr = st.test_round(nv, np.stack(rows), gl, gt, lw, gw, 1.0)
            got = [(gt[int(r["group"])], int(r["engine_id"]), int(r["lane_mask"])) for r in recs]
            assert got == reps, (name, k)
            assert [len(recs), ctr["clauses_tested"], len(rows), ctr["aggregate_tests_negative"]] == result, (name, k)
        if gw < 32:
            assert multi > 0, name  # the narrow fixture has multi-chunk rounds
