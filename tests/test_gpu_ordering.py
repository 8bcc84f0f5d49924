"""Device-side ordering of a round's records (tsg_fetch_ordered, hand-written
LSD radix sort, tsg_sort.cuh) against the host ordering of the same records
(reports.reference_order, numpy lexsort): destination-major, then chunk,
bucket creation rank, engine id, group -- the reference's delivery order
(engine.py:403-414, 462-464) -- at sizes where the sort runs many blocks and
every key width is exercised; small rounds take the host-sort path of the
same call."""
import ctypes as C

import numpy as np
import pytest

from gpu_util import require_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,nv,threads,lanes,lw,gw,rec", [
    (200_000, 3000, 4, 32, 32, 32, 8),      # 8-byte kernel records
    (200_000, 3000, 5, 70, 32, 4, 16),      # 16-byte records, 3 chunks, threads spanning chunks
    (60_000, 500, 3, 90, 64, 64, 16),       # 64-bit lane masks
    (2_000_000, 50_000, 8, 32, 32, 32, 8),  # C2-sized store
    # small rounds (<= 16384 records): keys from the device, sorted on the host
    (20_000, 2000, 3, 32, 32, 32, 8),
    (20_000, 2000, 3, 40, 32, 4, 16),
    (8_000, 500, 2, 70, 64, 64, 16),
    # 1200 one-lane groups: 19 chunks, wide chunk and group fields (both paths)
    (60_000, 600, 4, 300, 1, 64, 16),
    (2_000, 600, 4, 300, 1, 64, 16),
])
def test_device_order_matches_host_order(n, nv, threads, lanes, lw, gw, rec):
    require_device()
    from paper_2012_03119_b200 import _lib
    from paper_2012_03119_b200 import reports as R
    from paper_2012_03119_b200 import workload as W
    from paper_2012_03119_b200.native import NativeEngine
    rng = np.random.default_rng(n + gw)
    buckets = W.clause_buckets(n, nv, rng, 1, 14)
    flat, offs, ids = W.flatten(buckets)
    e = NativeEngine(nv, lw, gw, report_capacity=1 << 16)
    if rec == 8:
        e.set_record_bytes(8)
    e.add_clauses(flat, offs, ids)
    snaps = W.snapshots(threads, lanes, nv, rng)
    gl, gt = W.groups_for(threads, lanes, lw)
    e.stage(snaps)
    r = e.round(gl, gt, 1.0)
    assert r.reports > 500
    # the bucket creation rank by size, shuffled: the order must follow the table passed in
    sizes = list(buckets)
    rank_of_size = np.zeros(max(sizes) + 1, np.int32)
    perm = rng.permutation(len(sizes))
    for k, s in enumerate(sizes):
        rank_of_size[s] = perm[k]
    eids = np.empty(r.reports, np.int64)
    masks = np.empty(r.reports, np.uint64)
    groups = np.empty(r.reports, np.int32)
    n_dest = len(np.unique(gt))
    counts = np.zeros(n_dest, np.int64)
    got = C.c_int64(0)
    hs = (C.c_void_p * 1)(e.h.value)
    _lib.check(e.L.tsg_fetch_ordered(hs, 1, _lib.ptr(rank_of_size), len(rank_of_size), _lib.ptr(eids), 8,
                                     _lib.ptr(masks), 8, _lib.ptr(groups), _lib.ptr(counts), r.reports,
                                     C.byref(got)))
    assert got.value == r.reports and counts.sum() == r.reports
    dec = e.fetch(r.reports)
    size_of = np.diff(offs)[dec["engine_id"] - ids[0]]
    order = np.lexsort((dec["group"], dec["engine_id"], rank_of_size[size_of], dec["group"] // gw,
                        gt[dec["group"]]))
    want = dec[order]
    assert np.array_equal(eids, want["engine_id"])
    assert np.array_equal(masks, want["lane_mask"])
    assert np.array_equal(groups, want["group"])
    assert np.array_equal(counts, np.bincount(gt[dec["group"]], minlength=n_dest))
    e.close()
