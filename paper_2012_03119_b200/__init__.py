"""B200-native GpuShareSat clause-usefulness filter (arXiv 2012.03119).

Drop-in for the hot path of the reference package `triggersat`: the
exchange engine (Engine, EngineConfig, Report, RoundResult, AssignmentSnapshot)
and the bit-parallel library (pack_assignments, build_aggregate_batch,
assignment_trigger, aggregate_trigger, multi_trigger).  Compute runs in the
hand-written sm_100a kernels of libtsg.so behind the C ABI in include/tsg.h.
"""
from ._lib import CapacityError, TsgError
from .bitpack import (
    FALSE,
    TRUE,
    UNDEF,
    AggregateAssignment,
    AggregateBatch,
    PackedAssignmentBatch,
    aggregate_trigger,
    aggregate_trigger_many,
    assignment_trigger,
    assignment_trigger_many,
    build_aggregate_batch,
    iter_set_bits,
    multi_trigger,
    pack_assignments,
)
from .engine import AssignmentSnapshot, Engine, EngineConfig, Report, RoundResult, RoundTrace
from .stats import EngineStats, stats_summary

__version__ = "0.1.0"

__all__ = [
    "TRUE", "FALSE", "UNDEF", "CapacityError", "TsgError",
    "PackedAssignmentBatch", "AggregateAssignment", "AggregateBatch",
    "pack_assignments", "assignment_trigger", "assignment_trigger_many",
    "build_aggregate_batch", "aggregate_trigger", "aggregate_trigger_many",
    "iter_set_bits", "multi_trigger",
    "Engine", "EngineConfig", "Report", "RoundResult", "RoundTrace", "AssignmentSnapshot",
    "EngineStats", "stats_summary", "__version__",
]
