"""C5 measurement: random 3-SAT near threshold, the
reference's CDCL solver threads exchanging clauses through (a) the
reference engine and (b) the GPU engine, same instance, seeds and time
budget.  Prints one JSON object per engine (imports per assignment, drop
ratio, negative-aggregate ratio, tests/s) -- PAPER.md:384-390 quantities.

    python tools/exchange_loop.py [n=20000] [threads=8] [seconds=60]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_03119_b200 import exchange as X  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 8
secs = float(sys.argv[3]) if len(sys.argv) > 3 else 60.0
if X.import_reference() is None:
    print(json.dumps({"unavailable": "reference package not installed (baseline/_ref)"}))
    sys.exit(0)
formula = X.random_3cnf(n, 4.26, 20121 + 5)
for gpu in (False, True):
    ans = X.run(formula, threads=threads, timeout=secs, seed=5, gpu=gpu)
    out = {"engine": "gpu (paper_2012_03119_b200)" if gpu else "reference (triggersat.engine)",
           "instance": f"random 3-SAT n={n} m={len(formula.clauses)} (ratio 4.26, seed {20121 + 5})",
           "threads": threads, "budget_s": secs}
    out.update(X.summary(ans))
    print(json.dumps(out), flush=True)
