"""World-size-2 gloo run of the row-sharded search plumbing (CPU only).

ShardedFlatIndex's shard split, global-row tagging, packing, all-gather and
merge order are exercised with the oracle as the local search and merge, and
the merged answer must equal the unsharded oracle answer — including a tie
group that straddles the shard boundary and a self-snap hit.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    rng = np.random.default_rng(31)
    n, d = 701, 24
    X = rng.normal(size=(n, d))
    X = (X / np.linalg.norm(X, axis=1, keepdims=True)).astype(np.float32)
    X[349] = X[10]   # rank 0 holds rows [0, 351): tie group straddles the split
    X[351] = X[10]
    X[700] = X[10]
    Q = rng.normal(size=(9, d))
    Q = (Q / np.linalg.norm(Q, axis=1, keepdims=True)).astype(np.float32)
    Q[4] = X[10]
    return X, Q


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import shard_merge
        from paper_2506_21593_b200.index import BatchResult
        from paper_2506_21593_b200.sharded import LocalHits, ShardedFlatIndex, shard_range

        X, Q = _data()
        lo, hi = shard_range(X.shape[0], rank, world)

        def local_search(q, k, mode):
            rows, raw, snap, count = shard_merge.local_hits(X[lo:hi], lo, q.numpy(), k)
            return LocalHits(torch.from_numpy(rows), torch.from_numpy(raw), torch.from_numpy(snap),
                             torch.from_numpy(count))

        def merge(parts, B, k):
            r, raw, rep, cnt = shard_merge.merge(
                [(p.rows.numpy(), p.raw.numpy(), p.snap.numpy(), p.count.numpy()) for p in parts], B, k)
            return BatchResult(torch.from_numpy(r), torch.from_numpy(rep), torch.from_numpy(raw),
                               torch.from_numpy(cnt))

        sh = ShardedFlatIndex(None, lo, local_search=local_search, merge=merge)
        res = sh.search_batch(torch.from_numpy(Q), 7)
        if rank == 0:
            np.savez(out_path, rows=res.rows.numpy(), raw=res.raw.numpy(), rep=res.scores.numpy(),
                     count=res.count.numpy())
    finally:
        dist.destroy_process_group()


def test_sharded_merge_equals_unsharded_gloo(tmp_path):
    import torch.multiprocessing as mp

    from oracle import flat_index as F

    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    X, Q = _data()
    want = F.search(X, Q, 7)
    np.testing.assert_array_equal(got["rows"], want.rows)
    np.testing.assert_array_equal(got["raw"], want.raw)
    np.testing.assert_array_equal(got["rep"], want.reported)
    np.testing.assert_array_equal(got["count"], want.count)
    assert list(got["rows"][4][:4]) == [10, 349, 351, 700]
