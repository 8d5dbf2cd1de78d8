"""Multi-rank device path on ONE GPU: 2, 3 and 4 ranks (processes) share cuda:0 and gloo
carries the collectives' CUDA tensors, so the code that runs per rank on an 8-GPU box —
the local tcgen05/exact scan, the snap flags (pr_index_snap_flags), the all-gather, the
device merge (pr_merge_shards), the hash-partitioned KV (pr_kv_*_owned + all-reduce) —
runs here exactly, only the transport differs from NCCL.

Checked against the unsharded index (bit-identical rows, raw and reported scores, counts)
and a dict oracle with last-write-wins (caches.py:57-77)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(n=240_000, d=256, B=384):
    rng = np.random.default_rng(71)
    X = rng.standard_normal((n, d), dtype=np.float32)
    X /= np.linalg.norm(X.astype(np.float64), axis=1, keepdims=True).astype(np.float32)
    Q = rng.standard_normal((B, d), dtype=np.float32)
    Q /= np.linalg.norm(Q.astype(np.float64), axis=1, keepdims=True).astype(np.float32)
    # near-duplicates, a self-snap query, and an exact-tie group straddling every shard
    # boundary of world 2/3/4 (rank r's first and last rows)
    Q[: B // 4] = X[rng.integers(0, n, B // 4)] + 0.05 * Q[: B // 4]
    Q[: B // 4] /= np.linalg.norm(Q[: B // 4].astype(np.float64), axis=1, keepdims=True).astype(np.float32)
    for w in (2, 3, 4):
        for r in range(1, w):
            lo = r * n // w
            X[lo - 1] = X[5]
            X[lo] = X[5]
    Q[B // 4] = X[5]
    return X, Q


def _index_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_21593_b200 import MODE_AUTO, MODE_EXACT, MODE_TENSOR, MODE_TENSOR_I8, FlatIndex
        from paper_2506_21593_b200.sharded import ShardedFlatIndex, shard_range

        X, Q = _data()
        n = X.shape[0]
        lo, hi = shard_range(n, rank, world)
        idx = FlatIndex(dim=X.shape[1], capacity=hi - lo)
        idx.extend_arrays([str(i) for i in range(lo, hi)], torch.from_numpy(X[lo:hi]).cuda(), validate=False)
        sh = ShardedFlatIndex(idx, lo)
        q = torch.from_numpy(Q).cuda()
        bad = {}
        full = None
        if rank == 0:
            full = FlatIndex(dim=X.shape[1], capacity=n)
            full.extend_arrays([str(i) for i in range(n)], torch.from_numpy(X).cuda(), validate=False)
        for mode in (MODE_AUTO, MODE_EXACT, MODE_TENSOR, MODE_TENSOR_I8):
            for k in (1, 5, 10):
                r = sh.search_batch(q, k, mode=mode)
                torch.cuda.synchronize()
                if rank == 0:
                    w = full.search_batch(q, k, mode=MODE_EXACT, validate=False)
                    bad[(mode, k)] = sum(int((a != b).sum().item()) for a, b in
                                         ((r.rows, w.rows), (r.raw, w.raw), (r.scores, w.scores), (r.count, w.count)))
        if rank == 0:
            np.save(out, np.array([[m, k, v] for (m, k), v in bad.items()]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_index_equals_single_index(gpu, tmp_path, world):
    import torch.multiprocessing as mp

    out = str(tmp_path / "bad.npy")
    mp.spawn(_index_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    bad = np.load(out)
    assert bad.shape[0] == 12
    assert (bad[:, 2] == 0).all(), bad


def _kv_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_21593_b200 import _lib
        from paper_2506_21593_b200.sharded_kv import ShardedKV, owner_host

        rng = np.random.default_rng(17)
        keys = [f"query-{i:09d}" for i in range(20000)] + ["Who wrote Hamlet?", "Who wrote Hamlet? ", "ünï ✓",
                                                            "x" * 70]
        kv = ShardedKV(capacity=40000)
        seq = 0
        for _ in range(3):
            puts = [keys[int(i)] for i in rng.integers(0, len(keys), 15000)]
            kv.put(puts, np.arange(seq, seq + len(puts)))
            seq += len(puts)
        probes = keys + [f"absent-{i}" for i in range(500)]
        vals, hit = kv.get(probes)
        live = int(_lib.load().pr_kv_size(kv._h, _lib.stream_ptr()))
        mine = sum(owner_host(k, world) == rank for k in set(keys))
        sizes = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([live], dtype=torch.int64, device="cuda"))
        if rank == 0:
            np.savez(out, vals=vals.cpu().numpy(), hit=hit.cpu().numpy(),
                     sizes=np.array([int(s.item()) for s in sizes]))
        assert live <= mine
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_kv_device_equals_dict(gpu, tmp_path, world):
    import torch.multiprocessing as mp

    out = str(tmp_path / "kv.npz")
    mp.spawn(_kv_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    rng = np.random.default_rng(17)
    keys = [f"query-{i:09d}" for i in range(20000)] + ["Who wrote Hamlet?", "Who wrote Hamlet? ", "ünï ✓", "x" * 70]
    want: dict = {}
    seq = 0
    for _ in range(3):
        for t in [keys[int(i)] for i in rng.integers(0, len(keys), 15000)]:
            want[t] = seq
            seq += 1
    probes = keys + [f"absent-{i}" for i in range(500)]
    exp = np.array([want.get(t, -1) for t in probes])
    np.testing.assert_array_equal(got["vals"], exp)
    np.testing.assert_array_equal(got["hit"], exp >= 0)
    sizes = got["sizes"]
    assert sizes.sum() == len(want)
    # ownership spreads the keys: every rank holds ~1/world of them
    assert sizes.min() > 0.8 * len(want) / world


def _cascade_kb(n_ctx=3000, n_dist=120_000, dim=384, seed=5):
    """(ids, payloads, vectors) of a knowledge base: HashEmbedder contexts of a synthetic
    QA pool + dense random distractors, and the pool's questions."""
    from benchlib.workloads import corpus_of, qa_rows
    from paper_2506_21593_b200 import HashEmbedder, Passage
    from paper_2506_21593_b200.vectors import EmbeddingVector

    emb = HashEmbedder(dim=dim)
    rows = qa_rows(n_ctx, seed=seed)
    corpus = corpus_of(rows)
    ctx = emb.embed_matrix([c["text"] for c in corpus]).astype(np.float32)
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((n_dist, dim), dtype=np.float32)
    D /= np.linalg.norm(D.astype(np.float64), axis=1, keepdims=True).astype(np.float32)
    X = np.concatenate([ctx, D])
    perm = rng.permutation(X.shape[0])  # contexts spread over every shard
    X = X[perm]
    base = [Passage(id=f"c{i}", text=c["text"], source=c["source"], embedding=EmbeddingVector(values=ctx[i]),
                    answer=c["answer"]) for i, c in enumerate(corpus)]
    base += [Passage(id=f"d{i}", text=f"distractor passage {i}", source="noise",
                     embedding=EmbeddingVector(values=D[i])) for i in range(n_dist)]
    payloads = [base[int(p)] for p in perm]
    return [p.id for p in payloads], payloads, X, [r["question"] for r in rows], emb


def _cascade_worker(rank, world, port, out, mode_name):
    import hashlib

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2506_21593_b200 as P
        from benchlib.workloads import simulate_batched
        from paper_2506_21593_b200.sharded import ShardedRowIndex, shard_range

        mode = getattr(P, mode_name)
        ids, payloads, X, questions, emb = _cascade_kb()
        lo, hi = shard_range(len(ids), rank, world)
        idx = ShardedRowIndex.load(ids, payloads, X[lo:hi], dim=X.shape[1])
        kb = P.MainKnowledgeBase.from_index(idx)
        router = P.CascadeRouter(embedder=emb, backend=P.StubBackend(), knowledge_base=kb)

        def route_all(r):
            logs = simulate_batched(r, questions, n_sessions=2, n_queries=700, seed=3, batch=256)
            # route_batch with an explicit mode (the KB scan path under test)
            qs = [P.validate_query(t, "m", query_id=f"m{i}") for i, t in enumerate(questions[:300] * 2)]
            r.reset_session()
            res = r.route_batch(qs, span=128, mode=mode)
            extra = [(a.text, a.layer.wire_name, a.supporting_passage_ids) for a, _ in res]
            return logs, extra, r.stats()

        logs, extra, st = route_all(router)
        digest = hashlib.sha256(repr((logs, extra, st)).encode()).hexdigest()
        ds = [None] * world
        dist.all_gather_object(ds, digest)
        if rank == 0:
            full = P.FlatIndex(dim=X.shape[1], capacity=len(ids))
            full.extend_arrays(ids, X, payloads=payloads, validate=False)
            ref = P.CascadeRouter(embedder=emb, backend=P.StubBackend(),
                                  knowledge_base=P.MainKnowledgeBase.from_index(full))
            want = route_all(ref)
            same = [a == b for a, b in zip(logs, want[0])] + [extra == want[1], st == want[2]]
            np.save(out, np.array([int(all(same)), int(len(set(ds)) == 1),
                                   sum(len(s) for s in logs), st["layer_counts"].get("naive_rag", 0)]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "MODE_AUTO"), (3, "MODE_TENSOR_I8"), (2, "MODE_EXACT")])
def test_route_batch_over_row_sharded_knowledge_base(gpu, tmp_path, world, mode):
    """The cascade with its knowledge base row-sharded over ranks (ShardedRowIndex: local
    scan + all-gather merge, seed and AKM rows gathered from their owning ranks) routes
    exactly like the single-GPU router: byte-identical session logs, answers, passages and
    counters on every rank."""
    import torch.multiprocessing as mp

    out = str(tmp_path / "casc.npy")
    mp.spawn(_cascade_worker, args=(world, _free_port(), out, mode), nprocs=world, join=True)
    same, ranks_agree, n, l5 = np.load(out)
    assert n == 1400 and l5 > 100
    assert ranks_agree == 1
    assert same == 1
