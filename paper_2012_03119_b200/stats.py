"""Engine statistics, same definitions as the reference
(instrumentation.py:203-258): clauses_tested_per_second = lane_tests /
busy_seconds, i.e. clause x assignment tests per second."""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional


@dataclass
class EngineStats:
    clauses_tested_per_second: Optional[float]
    assignment_drop_ratio: Optional[float]
    negative_aggregate_ratio: Optional[float]
    imports_per_assignment: Optional[float]
    store_size: int
    zero_denominators: tuple = ()

    def as_dict(self) -> dict:
        return {
            "clauses_tested_per_second": self.clauses_tested_per_second,
            "assignment_drop_ratio": self.assignment_drop_ratio,
            "negative_aggregate_ratio": self.negative_aggregate_ratio,
            "imports_per_assignment": self.imports_per_assignment,
            "store_size": self.store_size,
            "zero_denominators": list(self.zero_denominators),
        }


def stats_summary(counters: dict) -> EngineStats:
    flags = []

    def ratio(num, den, name):
        if den <= 0:
            flags.append(name)
            return None
        return num / den

    negative = ratio(counters.get("aggregate_tests_negative", 0), counters.get("aggregate_tests", 0),
                     "negative_aggregate_ratio")
    submitted = counters.get("snapshots_accepted", 0) + counters.get("snapshots_dropped", 0)
    drop = ratio(counters.get("snapshots_dropped", 0), submitted, "assignment_drop_ratio")
    imports = ratio(counters.get("reports_delivered", 0), counters.get("snapshots_consumed", 0),
                    "imports_per_assignment")
    tested = ratio(counters.get("lane_tests", 0), counters.get("busy_seconds", 0.0),
                   "clauses_tested_per_second")
    return EngineStats(clauses_tested_per_second=tested, assignment_drop_ratio=drop,
                       negative_aggregate_ratio=negative, imports_per_assignment=imports,
                       store_size=counters.get("store_size", 0), zero_denominators=tuple(flags))
