"""The clause-exchange loop with the reference's CDCL solver threads
(SURVEY.md §8(d) C5, §8(f)2): `solve_parallel` of the reference
orchestrator (orchestrator.py:84-198) with this package's GPU Engine in
place of triggersat.engine.Engine -- the injection seam is the `Engine`
symbol the orchestrator constructs (orchestrator.py:18, 91-100); the solver
side (solver.py:383-541) is the reference's, unchanged.

The reference package is a caller here, not part of the product: it is
imported from `baseline/_ref` (pip --target install of /root/reference,
DESIGN.md §8) or from an importable `triggersat`.
"""
from __future__ import annotations

import contextlib
import os
import sys
from typing import Optional

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def import_reference():
    """The reference package (triggersat), or None when it is not installed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "triggersat")) and ref not in sys.path:
        sys.path.append(ref)
    try:
        import triggersat  # noqa: F401
        import triggersat.orchestrator  # noqa: F401
        return triggersat
    except ImportError:
        return None


def random_3cnf(num_vars: int, ratio: float, seed: int):
    """Uniform random 3-SAT, m = round(ratio * n) clauses of 3 distinct
    variables with random signs (the recipe of the reference's
    tests/oracles.py:110-118)."""
    ts = import_reference()
    rng = np.random.default_rng(seed)
    m = int(round(ratio * num_vars))
    clauses = []
    for _ in range(m):
        vs = rng.choice(num_vars, 3, replace=False) + 1
        sg = rng.integers(0, 2, 3) * 2 - 1
        clauses.append([int(v * s) for v, s in zip(vs, sg)])
    return ts.core.Formula(num_vars, clauses)


@contextlib.contextmanager
def gpu_engine_in_orchestrator(trace: bool = False, device: int = 0, keep: Optional[list] = None):
    """Within the block, the reference orchestrator builds this package's GPU
    Engine.  `keep` (a list) receives every engine built, for inspection."""
    ts = import_reference()
    from . import engine as E
    orch = ts.orchestrator
    saved = (orch.Engine, orch.EngineConfig)

    def make_engine(num_vars, threads, cfg):
        eng = E.Engine(num_vars, threads, E.EngineConfig(
            max_clauses=cfg.max_clauses, lane_width=cfg.lane_width, group_width=cfg.group_width,
            trace=trace, device=device))
        if keep is not None:
            keep.append(eng)
        return eng

    orch.Engine = make_engine
    try:
        yield
    finally:
        orch.Engine, orch.EngineConfig = saved


def run(formula, threads: int = 4, timeout: float = 60.0, seed: int = 0, gpu: bool = True,
        trace: bool = False, keep: Optional[list] = None):
    """One solve_parallel run; returns the reference's FinalAnswer."""
    ts = import_reference()
    cfg = ts.orchestrator.RunConfig(threads=threads, timeout=timeout, seed=seed)
    if not gpu:
        return ts.orchestrator.solve_parallel(formula, cfg)
    with gpu_engine_in_orchestrator(trace=trace, keep=keep):
        return ts.orchestrator.solve_parallel(formula, cfg)


def summary(ans) -> dict:
    """Exchange statistics of a run (instrumentation.py:228-258 plus solver imports)."""
    st = ans.engine_stats
    imports = sum(s.get("imports_attached", 0) + s.get("imports_implied", 0) + s.get("imports_conflict", 0)
                  for s in ans.solver_stats)
    return {
        "status": ans.status.value, "wall_s": ans.wall_time,
        "conflicts": sum(s.get("conflicts", 0) for s in ans.solver_stats),
        "snapshots_submitted": sum(s.get("snapshots_submitted", 0) for s in ans.solver_stats),
        "clauses_exported": sum(s.get("exported", 0) for s in ans.solver_stats),
        "reports_drained": sum(s.get("reports_drained", 0) for s in ans.solver_stats),
        "clauses_imported": imports,
        "imports_per_assignment": st.imports_per_assignment if st else None,
        "assignment_drop_ratio": st.assignment_drop_ratio if st else None,
        "negative_aggregate_ratio": st.negative_aggregate_ratio if st else None,
        "clauses_tested_per_second": st.clauses_tested_per_second if st else None,
        "engine_rounds": ans.engine_counters.get("rounds") if ans.engine_counters else None,
    }
