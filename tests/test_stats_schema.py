"""stats_summary / EngineStats against the reference's own
(instrumentation.py:203-258) on random counter dicts, zero denominators
included: identical fields, values and flag order.  Uses the installed
reference package (baseline/_ref) when present."""
import numpy as np
import pytest


def test_stats_match_reference():
    from paper_2012_03119_b200 import exchange as X
    from paper_2012_03119_b200.stats import stats_summary
    if X.import_reference() is None:
        pytest.skip("reference package not installed (baseline/_ref)")
    from triggersat.instrumentation import stats_summary as ref_summary
    rng = np.random.default_rng(3)
    keys = ("aggregate_tests_negative", "aggregate_tests", "snapshots_dropped", "snapshots_accepted",
            "reports_delivered", "snapshots_consumed", "lane_tests", "store_size")
    for _ in range(300):
        c = {k: int(rng.integers(0, 3) * rng.integers(0, 10 ** 6)) for k in keys if rng.random() < 0.9}
        c["busy_seconds"] = float(rng.choice([0.0, rng.random()]))
        assert stats_summary(c).as_dict() == ref_summary(c).as_dict(), c
