"""World-size-2 gloo run of the hash-partitioned KV plumbing (CPU only).

Each rank holds only the keys it owns (a dict stands in for the device table;
ownership uses the library's host fingerprint, i.e. the same bits the device
path uses), lookups are combined with one all-reduce(max), and the result must
equal a single unsharded dict with last-write-wins.
"""
from __future__ import annotations

import os
import socket

import numpy as np


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _script():
    rng = np.random.default_rng(9)
    keys = [f"query-{i:09d}" for i in range(400)] + ["Who wrote Hamlet?", "Who wrote Hamlet? ", "ünï"]
    puts = [keys[int(i)] for i in rng.integers(0, len(keys), 900)]
    probes = keys + [f"absent-{i}" for i in range(50)]
    return puts, probes


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_21593_b200.sharded_kv import ShardedKV, owner_host

        table: dict[str, int] = {}

        def own(t):
            return owner_host(t, world)

        def insert(texts, vals, r, w):
            n = 0
            for t, v in zip(texts, vals.tolist()):
                if own(t) == r:
                    table[t] = max(table.get(t, -1), v)
                    n += 1
            return n

        def probe(texts, r, w):
            return torch.tensor([table.get(t, -1) for t in texts], dtype=torch.int64)

        kv = ShardedKV(probe=probe, insert=insert)
        puts, probes = _script()
        kv.put(puts, np.arange(len(puts)))
        vals, hit = kv.get(probes)
        if rank == 0:
            np.savez(out, vals=vals.numpy(), hit=hit.numpy(), mine=len(table))
    finally:
        dist.destroy_process_group()


def test_sharded_kv_equals_single_table(tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "kv.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    puts, probes = _script()
    want = {}
    for i, t in enumerate(puts):
        want[t] = i  # last write wins
    exp = np.array([want.get(t, -1) for t in probes])
    np.testing.assert_array_equal(got["vals"], exp)
    np.testing.assert_array_equal(got["hit"], exp >= 0)
    assert 0 < int(got["mine"]) < len(set(puts))  # rank 0 owns a strict subset


def test_owner_bits_disjoint_from_bucket_bits():
    """Round-1 bug: ownership and home bucket came from the same low fingerprint bits, so a
    rank's keys could only use 1/world of its buckets.  Owner now comes from the tag's high
    half and the bucket from the second word: every rank's keys spread over all buckets."""
    from paper_2506_21593_b200.caches import fingerprint_host
    from paper_2506_21593_b200.sharded_kv import owner_host

    world, nb = 8, 1 << 10
    buckets = [set() for _ in range(world)]
    for i in range(40000):
        t = f"query-{i:09d}"
        buckets[owner_host(t, world)].add(fingerprint_host(t)[1] & (nb - 1))
    for b in buckets:
        assert len(b) > 0.95 * nb
