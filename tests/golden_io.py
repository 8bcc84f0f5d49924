"""Loaders for the committed golden fixtures (produced by tests/golden/make_golden.py
from the reference implementation itself)."""
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bitpack_golden():
    with open(os.path.join(GOLDEN, "bitpack_golden.json")) as fh:
        return json.load(fh)


def engine_golden():
    with open(os.path.join(GOLDEN, "engine_golden.json")) as fh:
        return json.load(fh)
