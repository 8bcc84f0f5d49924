"""Logical conventions of the reference (core.py:5-45): values and literals.

TRUE=1, FALSE=-1, UNDEF=0; a literal is +v or -v for v in 1..num_vars; an
assignment is indexed by variable with slot 0 unused.  These are data
conventions shared with the solver threads, not compute.
"""
from __future__ import annotations

TRUE = 1
FALSE = -1
UNDEF = 0

VALUE_NAMES = {TRUE: "T", FALSE: "F", UNDEF: "U"}


def negate_value(w: int) -> int:
    return -w


def lit_var(lit: int) -> int:
    return lit if lit > 0 else -lit


def all_undef(num_vars: int) -> list:
    return [UNDEF] * (num_vars + 1)


def assignment_from_dict(num_vars: int, mapping: dict) -> list:
    values = [UNDEF] * (num_vars + 1)
    for var, w in mapping.items():
        values[var] = w
    return values
