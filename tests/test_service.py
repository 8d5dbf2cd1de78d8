"""Service micro-batching: MicroBatcher coalesces concurrent
route() calls into route_batch() and returns what sequential route() calls in
the served order would (reference POST /query, src/service.py:95-100)."""
from __future__ import annotations

import json
import os
import threading

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


class _FakeError(Exception):
    pass


def _fake_batcher(**kw):
    from paper_2506_21593_b200.errors import AllLayersMissed
    from paper_2506_21593_b200.service import MicroBatcher

    sizes = []

    def batch_fn(queries):
        sizes.append(len(queries))
        return [AllLayersMissed(f"miss {q}") if q % 5 == 0 else ("answer", q) for q in queries]

    b = MicroBatcher(router=None, batch_fn=batch_fn, record_order=True, **kw)
    return b, sizes


def test_concurrent_requests_share_batches_and_get_their_own_results():
    from paper_2506_21593_b200.errors import AllLayersMissed

    b, sizes = _fake_batcher(max_batch=64, max_wait_s=0.02)
    out = {}
    barrier = threading.Barrier(40)

    def client(i):
        barrier.wait()
        try:
            out[i] = b.route(i, timeout=10)
        except AllLayersMissed as exc:  # the per-request error of router.route
            out[i] = str(exc)

    ts = [threading.Thread(target=client, args=(i,)) for i in range(1, 41)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    b.close()
    assert len(out) == 40
    for i in range(1, 41):
        assert out[i] == (f"miss {i}" if i % 5 == 0 else ("answer", i))
    assert sum(sizes) == 40 and len(sizes) < 40  # coalesced
    assert sorted(b.served_order) == list(range(1, 41))


def test_max_batch_and_close_drains():
    b, sizes = _fake_batcher(max_batch=3, max_wait_s=0.05)
    futs = [b.submit(i) for i in range(1, 11)]
    b.close()
    assert all(f.done() for f in futs)
    assert max(sizes) <= 3 and sum(sizes) == 10
    with pytest.raises(RuntimeError):
        b.submit(99)


def test_batch_failure_reaches_every_waiter():
    from paper_2506_21593_b200.service import MicroBatcher

    def boom(queries):
        raise _FakeError("device lost")

    b = MicroBatcher(router=None, batch_fn=boom)
    f = b.submit(1)
    with pytest.raises(_FakeError):
        f.result(timeout=5)
    b.close()


@pytest.mark.gpu
def test_micro_batched_router_equals_sequential_routes(gpu):
    from paper_2506_21593_b200 import CascadeRouter, HashEmbedder, StubBackend, ingest_corpus, validate_query
    from paper_2506_21593_b200.service import MicroBatcher

    with open(os.path.join(HERE, "golden", "router_trace.json")) as fh:
        gold = json.load(fh)

    def router():
        emb = HashEmbedder()
        kb = ingest_corpus((json.dumps(c) for c in gold["corpus"]), emb)
        return CascadeRouter(embedder=emb, backend=StubBackend(), knowledge_base=kb)

    texts = [q["text"] for q in gold["queries"]]
    qs = [validate_query(t, "s1", query_id=f"q{i}", issued_at_ns=i) for i, t in enumerate(texts)]
    live = router()
    got = {}
    with MicroBatcher(live, max_batch=32, max_wait_s=0.002, record_order=True) as b:
        def client(lo):
            for q in qs[lo::8]:
                got[q.id] = b.route(q, timeout=60)

        ts = [threading.Thread(target=client, args=(i,)) for i in range(8)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        order = list(b.served_order)
        assert b.batches < len(qs)
    twin = router()
    for q in order:
        a, ev = twin.route(q)
        a2, ev2 = got[q.id]
        assert (a2.text, a2.layer, list(a2.supporting_passage_ids)) == (a.text, a.layer, list(a.supporting_passage_ids))
        assert [(p.layer, p.outcome) for p in ev2.layers_probed] == [(p.layer, p.outcome) for p in ev.layers_probed]
    assert live.stats()["layer_counts"] == twin.stats()["layer_counts"]
