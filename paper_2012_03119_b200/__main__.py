"""`python -m paper_2012_03119_b200 FILE.cnf [flags]` -- the reference's own
command line (cli.py:126-241: DIMACS in, SAT-competition answer and exit
code 10/20/0 out, `--stats-json` with the engine statistics of
instrumentation.py:203-258) with this package's GPU engine in its clause
exchange.  The CLI and solver are the reference's,
imported from baseline/_ref (exchange.py)."""
from __future__ import annotations

import sys

from .exchange import gpu_engine_in_orchestrator, import_reference


def main(argv=None) -> int:
    if import_reference() is None:
        print("the reference package (triggersat) is not installed (baseline/_ref)", file=sys.stderr)
        return 1
    import triggersat.cli as cli
    with gpu_engine_in_orchestrator():
        return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
