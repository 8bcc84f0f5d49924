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


def c5_replays():
    """{name: loaded npz} of the reference solver's recorded exchange rounds
    (tests/golden/make_c5_replay.py)."""
    import numpy as np
    out = {}
    for f in sorted(os.listdir(GOLDEN)):
        if f.startswith("c5_replay_") and f.endswith(".npz"):
            out[f[len("c5_replay_"):-4]] = dict(np.load(os.path.join(GOLDEN, f)))
    return out


def c5_round(fx, k):
    """Round k of a C5 replay: (clause lits by engine id for ids < n_inserted,
    live ids, snapshots [(tid, values)], reports [(dest, eid, mask)] in emission
    order, RoundResult fields)."""
    off, lits = fx["ins_off"], fx["ins_lits"]
    n = int(fx[f"r{k}_n_inserted"])
    clauses = [tuple(int(x) for x in lits[off[i]:off[i + 1]]) for i in range(n)]
    snaps = list(zip(fx[f"r{k}_snap_tid"].tolist(), fx[f"r{k}_snap_vals"]))
    reps = list(zip(fx[f"r{k}_rep_dest"].tolist(), fx[f"r{k}_rep_eid"].tolist(), fx[f"r{k}_rep_mask"].tolist()))
    return clauses, set(fx[f"r{k}_live"].tolist()), snaps, reps, fx[f"r{k}_result"].tolist()
