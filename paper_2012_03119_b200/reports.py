"""Report records of the C ABI (include/tsg.h tsg_report, 16 bytes; 12- and
8-byte egress forms).

key = engine_id << 16 | group; lane_mask.  Helpers to decode, build and order
them the way the reference emits reports (engine.py:403-464): by chunk
(group // group_width), then creation rank of the clause's size bucket, then
slot -- which equals engine-id order inside a bucket, because clauses are
appended in id order and compaction preserves order (engine.py:150-163,
184-200) -- then group.
"""
from __future__ import annotations

from typing import Dict, Mapping

import numpy as np

RECORD_DTYPE = np.dtype([("key", "<u8"), ("lane_mask", "<u8")])
# 12-byte egress records (tsg_set_record_bytes(h, 12), lane_width <= 32)
RECORD12_DTYPE = np.dtype({"names": ["key", "lane_mask"], "formats": ["<u8", "<u4"], "offsets": [0, 8],
                           "itemsize": 12})
# 8-byte egress records (tsg_set_record_bytes(h, 8)): engine_id << 37 | group << 32 | lane_mask
RECORD8_DTYPE = np.dtype([("packed", "<u8")])
PAD_KEY = np.uint64(0xFFFFFFFFFFFFFFFF)
DECODED_DTYPE = np.dtype([("engine_id", "<i8"), ("group", "<i4"), ("lane_mask", "<u8")])


def decode(recs: np.ndarray) -> np.ndarray:
    out = np.zeros(len(recs), DECODED_DTYPE)
    if recs.dtype.names == ("packed",):
        p = recs["packed"]
        out["engine_id"] = (p >> np.uint64(37)).astype(np.int64)
        out["group"] = ((p >> np.uint64(32)) & np.uint64(31)).astype(np.int32)
        out["lane_mask"] = p & np.uint64(0xFFFFFFFF)
        return out
    out["engine_id"] = (recs["key"] >> np.uint64(16)).astype(np.int64)
    out["group"] = (recs["key"] & np.uint64(0xFFFF)).astype(np.int32)
    out["lane_mask"] = recs["lane_mask"]
    return out


def encode(engine_id, group, lane_mask) -> np.ndarray:
    out = np.zeros(len(engine_id), RECORD_DTYPE)
    out["key"] = (np.asarray(engine_id, np.uint64) << np.uint64(16)) | np.asarray(group, np.uint64)
    out["lane_mask"] = np.asarray(lane_mask, np.uint64)
    return out


def reference_order(dec: np.ndarray, group_width: int, bucket_rank: np.ndarray) -> np.ndarray:
    """Permutation putting decoded records in the reference's emission order.
    `bucket_rank[i]` is the creation rank of record i's size bucket."""
    grp = dec["group"].astype(np.int64)
    return np.lexsort((grp, dec["engine_id"], np.asarray(bucket_rank, np.int64), grp // group_width))


def bucket_ranks(dec: np.ndarray, size_of: Mapping[int, int], rank_of_size: Dict[int, int]) -> np.ndarray:
    return np.fromiter((rank_of_size[size_of[int(e)]] for e in dec["engine_id"]), dtype=np.int64,
                       count=len(dec))
