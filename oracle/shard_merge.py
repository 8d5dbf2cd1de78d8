"""TEST INFRASTRUCTURE ONLY — CPU restatement of the all-gather merge.

Merging per-shard exact top-k lists of a row-sharded FlatIndex must give the
unsharded FlatIndex.search answer (index.py:176: score desc, row asc; the
self-snap of index.py:180-181 is decided by the shard that owns the row).
Used by tests/test_sharded_gloo.py as the merge + local search of the CPU
(gloo) run of paper_2506_21593_b200.sharded.ShardedFlatIndex.
"""
from __future__ import annotations

import numpy as np

from . import flat_index as F


def local_hits(X_local: np.ndarray, row_offset: int, Q: np.ndarray, k: int):
    """Exact local top-k with GLOBAL row ids and per-hit snap flags."""
    res = F.search(X_local, Q, k)
    rows = np.where(res.rows >= 0, res.rows + row_offset, -1)
    snap = np.zeros(res.rows.shape, dtype=np.uint8)
    for b in range(res.rows.shape[0]):
        for j in range(int(res.count[b])):
            r = int(res.rows[b, j])
            snap[b, j] = res.raw[b, j] > 1.0 - 1e-6 and bool(np.array_equal(X_local[r], Q[b]))
    return rows, res.raw, snap, res.count


def merge(parts, B: int, k: int):
    """parts: list of (rows, raw, snap, count) per shard -> (rows, raw, reported, count)."""
    out_rows = np.full((B, k), -1, dtype=np.int64)
    out_raw = np.zeros((B, k))
    out_rep = np.zeros((B, k))
    out_cnt = np.zeros(B, dtype=np.int32)
    for b in range(B):
        cand = []
        for rows, raw, snap, count in parts:
            for j in range(int(count[b])):
                cand.append((-raw[b, j], int(rows[b, j]), bool(snap[b, j])))
        cand.sort()
        take = min(k, len(cand))
        out_cnt[b] = take
        for j in range(take):
            s, r, sn = -cand[j][0], cand[j][1], cand[j][2]
            out_rows[b, j] = r
            out_raw[b, j] = s
            out_rep[b, j] = 1.0 if sn else max(-1.0, min(1.0, s))
    return out_rows, out_raw, out_rep, out_cnt
