"""CPU-side checks of the C ABI: the in-tree library loads without a GPU and
exports every entry point include/tsg.h declares; without a device the
product fails loudly instead of falling back to a CPU path."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tsg.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(tsg_[a-z_0-9]+)\s*\(", src, re.M)))


def test_header_declares_the_bound_symbols():
    from paper_2012_03119_b200 import _lib
    assert set(header_symbols()) == set(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    from paper_2012_03119_b200 import _lib
    L = _lib.load()
    for name in header_symbols():
        assert hasattr(L, name), name
    assert L.tsg_abi_version() == 2


def test_no_cpu_fallback_without_device():
    from paper_2012_03119_b200 import _lib
    import paper_2012_03119_b200 as P
    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(P.TsgError):
        P.Engine(10, 2)
    with pytest.raises(P.TsgError):
        P.pack_assignments([[0, 1]], 1, 8)


def test_host_side_validation_matches_reference():
    import paper_2012_03119_b200 as P
    with pytest.raises(ValueError):
        P.EngineConfig(max_clauses=0)
    with pytest.raises(ValueError):
        P.EngineConfig(activity_decay=0.0)
    with pytest.raises(ValueError):
        P.EngineConfig(reduce_keep_fraction=1.0)
    with pytest.raises(ValueError):
        P.EngineConfig(assignment_queue_capacity=0)
    assert P.EngineConfig(lane_width=8).assignment_queue_capacity == 16
    with pytest.raises(P.CapacityError):
        P.pack_assignments([[0, 0]] * 3, 1, lane_width=2)
    with pytest.raises(ValueError):
        P.pack_assignments([], 1, lane_width=65)


@pytest.mark.parametrize("num_vars", [0, 1, 30, 31, 32, 63, 95, 1000, 4097])
def test_pack_rows_host_encoding(num_vars):
    # tsg_pack_rows is host code (snapshot ingress): 2 bits per variable,
    # low half (value == 1), high half (value != 0) -- bitpack.py:104-111
    from paper_2012_03119_b200.native import pack_rows, packed_words
    rng = np.random.default_rng(num_vars)
    rows = rng.choice(np.array([1, -1, 0, 0, 1, 5, -7], np.int8), size=(9, num_vars + 1 + 3))
    got = pack_rows(rows[:, :num_vars + 1], num_vars, threads=3)
    w = packed_words(num_vars)
    assert got.shape == (9, w) and w % 4 == 0 and 32 * w >= num_vars + 2
    t = np.zeros((9, 32 * w), bool)
    s = np.zeros((9, 32 * w), bool)
    t[:, :num_vars + 1] = rows[:, :num_vars + 1] == 1
    s[:, :num_vars + 1] = rows[:, :num_vars + 1] != 0
    bit = np.uint64(1) << np.arange(32, dtype=np.uint64)
    want = (t.reshape(9, w, 32) * bit).sum(2).astype(np.uint64) | \
        ((s.reshape(9, w, 32) * bit).sum(2).astype(np.uint64) << np.uint64(32))
    assert np.array_equal(got, want)


def test_ring_entry_points_validate_without_a_device():
    # the report ring's host-side argument checks (include/tsg.h tsg_ring_*)
    # need no GPU: a null handle or a missing ring is TSG_EINVAL
    import ctypes as C
    from paper_2012_03119_b200 import _lib
    L = _lib.load()
    n = C.c_int64(0)
    assert L.tsg_ring_drain(None, None, 0, C.byref(n), 0, None) == _lib.TSG_EINVAL
    assert L.tsg_ring_status(None, None, None, None) == _lib.TSG_EINVAL
    assert L.tsg_ring_open(None, 1024, 1000) == _lib.TSG_EINVAL
    assert L.tsg_ring_close(None) == _lib.TSG_EINVAL
