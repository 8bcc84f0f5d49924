"""Derived engine statistics with the reference's schema and definitions
(instrumentation.py:203-258): every statistic is a ratio of the engine's
counters (engine.py:284-299, raw_counters), None when its denominator is
zero, and the names of those are listed in `zero_denominators`.  The
headline, clauses_tested_per_second = lane_tests / busy_seconds, is the
clause x assignment test rate of run_round (instrumentation.py:248-250)."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, Optional, Tuple

# (statistic, numerator, denominator) over a counter dict, in the order the
# reference evaluates them (which fixes the order of zero_denominators)
_RATIOS: Tuple[Tuple[str, Callable[[dict], float], Callable[[dict], float]], ...] = (
    ("negative_aggregate_ratio", lambda c: c.get("aggregate_tests_negative", 0), lambda c: c.get("aggregate_tests", 0)),
    ("assignment_drop_ratio", lambda c: c.get("snapshots_dropped", 0),
     lambda c: c.get("snapshots_accepted", 0) + c.get("snapshots_dropped", 0)),
    ("imports_per_assignment", lambda c: c.get("reports_delivered", 0), lambda c: c.get("snapshots_consumed", 0)),
    ("clauses_tested_per_second", lambda c: c.get("lane_tests", 0), lambda c: c.get("busy_seconds", 0.0)),
)
_FIELDS = ("clauses_tested_per_second", "assignment_drop_ratio", "negative_aggregate_ratio",
           "imports_per_assignment", "store_size", "zero_denominators")


@dataclass
class EngineStats:
    clauses_tested_per_second: Optional[float]
    assignment_drop_ratio: Optional[float]
    negative_aggregate_ratio: Optional[float]
    imports_per_assignment: Optional[float]
    store_size: int
    zero_denominators: tuple = field(default=())

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k in _FIELDS}
        d["zero_denominators"] = list(self.zero_denominators)
        return d


def stats_summary(counters: dict) -> EngineStats:
    values: Dict[str, Optional[float]] = {}
    zero = []
    for name, num, den in _RATIOS:
        d = den(counters)
        if d > 0:
            values[name] = num(counters) / d
        else:
            values[name] = None
            zero.append(name)
    return EngineStats(store_size=counters.get("store_size", 0), zero_denominators=tuple(zero), **values)
