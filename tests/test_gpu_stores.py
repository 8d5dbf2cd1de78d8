"""Device stores and the router against the reference's recorded behaviour.

Golden replays (tests/golden, produced by the real reference) plus the
reference's unit-test scenarios (pkg/tests/test_caches.py, test_knowledge.py,
test_router.py) restated against the GPU drop-ins.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import random_unit_vectors

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _golden(name):
    with open(os.path.join(HERE, "golden", name)) as fh:
        return json.load(fh)


def ans(text="forty-two", layer=None):
    from paper_2506_21593_b200 import AnswerRecord, LayerTag

    layer = layer or LayerTag.NAIVE_RAG
    ps = ("p1",) if layer in (LayerTag.ADAPTIVE_MEMORY, LayerTag.NAIVE_RAG) else ()
    return AnswerRecord(text=text, layer=layer, confidence=0.9, supporting_passage_ids=ps)


# ---------------------------------------------------------------- FlatIndex golden
def test_flat_index_golden_both_paths(gpu):
    import torch

    from paper_2506_21593_b200 import MODE_AUTO, MODE_EXACT, MODE_TENSOR, FlatIndex

    meta = _golden("flat_index.json")["flat_index_cases"]
    g = np.load(os.path.join(HERE, "golden", "flat_index.npz"))
    for c in meta:
        nm = c["name"]
        X, Q, k = g[f"{nm}_X"], g[f"{nm}_Q"], c["k"]
        idx = FlatIndex(dim=c["d"])
        idx.extend_arrays([f"e{i}" for i in range(X.shape[0])], X)
        for mode in (MODE_EXACT, MODE_TENSOR, MODE_AUTO):
            res = idx.search_batch(torch.from_numpy(Q), k, mode=mode)
            cnt = res.count.cpu().numpy()
            np.testing.assert_array_equal(cnt, g[f"{nm}_count"])
            for b in range(Q.shape[0]):
                n = cnt[b]
                np.testing.assert_array_equal(res.rows.cpu().numpy()[b, :n], g[f"{nm}_rows"][b, :n], err_msg=nm)
                np.testing.assert_array_equal(res.scores.cpu().numpy()[b, :n], g[f"{nm}_scores"][b, :n], err_msg=nm)


# ---------------------------------------------------------------- fixed KV
def test_kv_golden_ops(gpu):
    from paper_2506_21593_b200 import AnswerRecord, FixedKVCache, LayerTag

    gold = _golden("kv_ops.json")
    kv = FixedKVCache(max_entries=gold["max_entries"])
    for op in gold["ops"]:
        if op["op"] == "put":
            kv.put(op["key"], AnswerRecord(text=op["value"], layer=LayerTag.MEMORY_RECALL, confidence=0.9))
        else:
            got = kv.get(op["key"])
            assert (got.text if got else None) == op["result"], op
        assert len(kv) == op["len"], op
    assert kv.stats() == gold["stats"]
    assert [e["query_text"] for e in kv.export_entries()] == gold["export"]


def test_kv_byte_exact_and_batch(gpu):
    from paper_2506_21593_b200 import FixedKVCache

    kv = FixedKVCache()
    kv.put("Who wrote Hamlet?", ans("Shakespeare"))
    assert kv.get("Who wrote Hamlet? ") is None
    assert kv.get("who wrote Hamlet?") is None
    assert kv.get("Who wrote Hamlet?").text == "Shakespeare"
    kv.put("Q1", ans("a1"))
    kv.put("Q1", ans("a2"))
    assert kv.get("Q1").text == "a2" and len(kv) == 2
    texts = [f"query-{i:09d}" for i in range(3000)]
    kv.put_many(texts + texts[:10], [ans(t) for t in texts] + [ans("late") for _ in range(10)])
    got = kv.get_batch(texts + ["absent", "Q1"])
    assert [g.text for g in got[:10]] == ["late"] * 10
    assert all(g.text == t for g, t in zip(got[10:3000], texts[10:]))
    assert got[3000] is None and got[3001].text == "a2"
    assert len(kv) == 3002


# ---------------------------------------------------------------- semantic cache
def test_semantic_cache_scenarios(gpu):
    from paper_2506_21593_b200 import HashEmbedder, SemanticCache, cosine

    emb = HashEmbedder()
    sc = SemanticCache(emb)
    sc.put("what is the tallest mountain", ans("everest"))
    rec, score = sc.lookup(emb.embed("what is the tallest mountain"))
    assert rec.text == "everest" and score == 1.0
    one = SemanticCache(emb, threshold=1.0)
    one.put("exact phrasing only", ans("yes"))
    assert one.lookup(emb.embed("exact phrasing only")) is not None
    # equality boundary is inclusive; next float above misses (test_caches.py:105-119)
    cached = "alpha beta gamma delta epsilon zeta eta theta iota"
    probe = "alpha beta gamma delta epsilon zeta eta theta kappa"
    s = cosine(emb.embed(cached), emb.embed(probe))
    at = SemanticCache(emb, threshold=s)
    at.put(cached, ans())
    assert at.lookup(emb.embed(probe)) is not None
    above = SemanticCache(emb, threshold=float(np.nextafter(s, 1.0)))
    above.put(cached, ans())
    assert above.lookup(emb.embed(probe)) is None
    # identical token bags tie exactly; the earlier insertion wins
    tie = SemanticCache(emb)
    tie.put("alpha beta gamma", ans("first"))
    tie.put("gamma beta alpha", ans("second"))
    rec, score = tie.lookup(emb.embed("beta alpha gamma"))
    assert score == 1.0 and rec.text == "first"
    # upsert keeps one row; eviction keeps most recent (test_caches.py:142-164)
    up = SemanticCache(emb)
    up.put("q", ans("old"))
    up.put("q", ans("new"))
    assert len(up) == 1 and up.lookup(emb.embed("q"))[0].text == "new"
    ev = SemanticCache(emb, max_entries=2)
    ev.put("first unique entry", ans("1"))
    ev.put("second unique entry", ans("2"))
    ev.put("first unique entry", ans("1b"))
    ev.put("third unique entry", ans("3"))
    assert len(ev) == 2
    assert ev.lookup(emb.embed("second unique entry")) is None
    assert ev.lookup(emb.embed("first unique entry"))[0].text == "1b"
    restored = SemanticCache.restore(up.snapshot(), emb)
    assert restored.lookup(emb.embed("q"))[0].text == "new"
    with pytest.raises(ValueError):
        SemanticCache(emb, threshold=0.0)


def test_semantic_lookup_batch_matches_single(gpu, rng):
    import torch

    from paper_2506_21593_b200 import HashEmbedder, SemanticCache

    emb = HashEmbedder(dim=768)
    sc = SemanticCache(emb, dim=768)
    X = random_unit_vectors(rng, 5000, 768)
    sc._index.extend_arrays([f"t{i}" for i in range(5000)], X,
                            payloads=[type("E", (), {"answer": ans(f"a{i}")})() for i in range(5000)])
    Q = random_unit_vectors(rng, 64, 768)
    Q[:20] = X[:20]
    hit, rows, scores = sc.lookup_batch(torch.from_numpy(Q))
    for b in range(64):
        single = sc.lookup(Q[b])
        assert bool(hit[b]) == (single is not None)
        if single is not None:
            assert single[1] == float(scores[b]) and sc.answer_at(int(rows[b])).text == single[0].text


# ---------------------------------------------------------------- knowledge
def test_knowledge_base_and_akm(gpu):
    from paper_2506_21593_b200 import (AdaptiveKnowledgeMemory, EmptyKnowledgeBase, HashEmbedder,
                                       MainKnowledgeBase, ingest_corpus)
    from oracle import flat_index as F

    emb = HashEmbedder()
    texts = [f"document about topic{i:02d} with body text {i}" for i in range(30)]
    lines = [json.dumps({"id": f"p{i}", "text": t, "source": "test"}) for i, t in enumerate(texts)]
    kb = ingest_corpus(lines, emb)
    assert len(kb) == 30 and "p3" in kb and kb.get("p3").source == "test"
    q = emb.embed("document about topic07")
    X = np.stack([kb.get(f"p{i}").embedding.values for i in range(30)])
    want = F.search(X, q.values[None, :], 10).rows[0]
    top, seeds = kb.retrieve(q, k=3, seed_k=10)
    assert [p.id for p in seeds] == [f"p{r}" for r in want]
    assert [p.id for p in top] == [p.id for p in seeds[:3]]
    with pytest.raises(EmptyKnowledgeBase):
        MainKnowledgeBase().retrieve(emb.embed("anything"), k=3)
    akm = AdaptiveKnowledgeMemory()
    akm.enqueue(seeds)
    assert len(akm) == 0 and akm.pending_count() == 10
    akm.settle()
    akm.enqueue(seeds)
    akm.settle()
    assert len(akm) == 10 and akm.inserted_total == 10
    assert akm.retrieve(emb.embed(seeds[0].text), k=3) is not None
    assert akm.retrieve(emb.embed("completely unrelated celestial navigation almanac"), k=3) is None
    restored = MainKnowledgeBase.restore(kb.snapshot())
    a, _ = kb.retrieve(q, k=3)
    b, _ = restored.retrieve(q, k=3)
    assert [p.id for p in a] == [p.id for p in b]


# ---------------------------------------------------------------- router golden replay
def _router_from_corpus(corpus, **kw):
    from paper_2506_21593_b200 import CascadeRouter, HashEmbedder, StubBackend, ingest_corpus

    emb = HashEmbedder()
    kb = ingest_corpus((json.dumps(c) for c in corpus), emb)
    return CascadeRouter(embedder=emb, backend=StubBackend(), knowledge_base=kb, **kw)


def test_router_matches_reference_trace(gpu):
    from paper_2506_21593_b200 import validate_query

    gold = _golden("router_trace.json")
    router = _router_from_corpus(gold["corpus"])
    for i, q in enumerate(gold["queries"]):
        if q["origin"] == "akm_probe":
            router.adaptive_memory.settle()
        answer, ev = router.route(validate_query(q["text"], "s1"))
        assert [[p.layer.wire_name, p.outcome] for p in ev.layers_probed] == q["probes"], i
        assert ev.serving_layer.wire_name == q["serving"], i
        assert answer.text == q["answer"], i
        assert list(answer.supporting_passage_ids) == q["passages"], i
    st = router.stats()
    g = gold["stats"]
    assert st["layer_counts"] == g["layer_counts"]
    assert st["fixed_kv"] == g["fixed_kv"]
    assert st["semantic_cache"] == g["semantic_cache"]
    assert st["adaptive_memory"] == g["adaptive_memory"]
    assert st["knowledge_base_searches"] == g["knowledge_base_searches"]
    assert router.semantic_cache.index.search_count == g["sc_searches"]
    assert router.adaptive_memory.index.search_count == g["akm_searches"]
    assert router.adaptive_memory.inserted_total == g["akm_inserted_total"]
    assert router.backend.context_calls == g["context_calls"]
    assert router.backend.recall_calls == g["recall_calls"]


def test_router_semantics(gpu):
    from paper_2506_21593_b200 import (AllLayersMissed, CascadeRouter, HashEmbedder, LayerTag, MainKnowledgeBase,
                                       RouterConfig, StubBackend, validate_query)

    gold = _golden("router_trace.json")
    router = _router_from_corpus(gold["corpus"])
    q0 = gold["queries"][0]["text"]
    router.route(validate_query(q0, "s1"))
    assert len(router.adaptive_memory) == 0 and router.adaptive_memory.pending_count() == 10
    before = (router.semantic_cache.index.search_count + router.adaptive_memory.index.search_count
              + router.knowledge_base.index.search_count)
    rep, ev = router.route(validate_query(q0, "s1"))
    after = (router.semantic_cache.index.search_count + router.adaptive_memory.index.search_count
             + router.knowledge_base.index.search_count)
    assert rep.layer is LayerTag.FIXED_KV and len(ev.layers_probed) == 1 and before == after
    assert rep.supporting_passage_ids == ()
    router.reset_session()
    assert len(router.kv_cache) == 0 and len(router.semantic_cache) == 0 and len(router.adaptive_memory) == 0
    cfg = RouterConfig(disabled_layers=frozenset({LayerTag.MEMORY_RECALL, LayerTag.ADAPTIVE_MEMORY}))
    r2 = _router_from_corpus(gold["corpus"], config=cfg)
    _, ev = r2.route(validate_query(q0, "s1"))
    assert [p.layer for p in ev.layers_probed] == [LayerTag.FIXED_KV, LayerTag.SEMANTIC_CACHE, LayerTag.NAIVE_RAG]
    empty = CascadeRouter(embedder=HashEmbedder(), backend=StubBackend(), knowledge_base=MainKnowledgeBase())
    with pytest.raises(AllLayersMissed) as err:
        empty.route(validate_query("anything at all", "s1"))
    assert err.value.trace_event.serving_layer is None
    assert len(empty.kv_cache) == 0 and len(empty.semantic_cache) == 0


def test_akm_settle_from_rows_mixed_paths(gpu):
    """settle_from_rows (device path, KB-row bitmap) interleaved with the host settle
    path, direct index inserts, clear and a knowledge-base that grows: the AKM holds
    exactly the ids the reference's settle would (first occurrence, no overwrite,
    knowledge.py:217-228), rows in insertion order, payloads = the KB passages."""
    from paper_2506_21593_b200 import AdaptiveKnowledgeMemory, HashEmbedder, Passage, ingest_corpus

    emb = HashEmbedder()
    lines = [json.dumps({"id": f"p{i}", "text": f"passage number {i} about subject {i % 7}", "source": "t"})
             for i in range(60)]
    kb = ingest_corpus(lines, emb)
    akm = AdaptiveKnowledgeMemory()
    want: list[str] = []

    def model_settle(ids):
        for pid in ids:
            if pid not in want:
                want.append(pid)

    rng = np.random.default_rng(5)
    for step in range(12):
        rows = rng.integers(0, len(kb), 25)
        if step == 3:  # host path: queued passages, some of them KB passages
            ps = [kb.get(f"p{r}") for r in rows[:6]]
            akm.enqueue(ps)
            akm.settle()
            model_settle([p.id for p in ps])
        if step == 5:  # an id inserted straight into the index
            p = kb.get("p59")
            akm.index.insert(p.id, p.embedding, p)
            model_settle([p.id])
        if step == 7:
            akm.clear()
            want.clear()
        if step == 9:  # the knowledge base grows: row marks are rebuilt
            for i in range(5):
                t = f"late passage {i}"
                kb.add(Passage(id=f"q{i}", text=t, source="t", embedding=emb.embed(t)))
        akm.settle_from_rows(kb.index, rows)
        model_settle([kb.index.id_at(int(r)) for r in rows])
        assert list(akm.index.entry_ids()) == want, step
        for pid in want[:5]:
            assert akm.index.payload(pid).id == pid


def test_deferred_payload_segments(gpu, rng):
    """append_rows_from without payloads defers each row's payload to the source row;
    truncate / clear / explicit appends / upserts interleave with it correctly."""
    from paper_2506_21593_b200 import FlatIndex

    d = 32
    X = random_unit_vectors(rng, 50, d)
    src = FlatIndex(dim=d)
    src.extend_arrays([f"s{i}" for i in range(50)], X, payloads=[("src", i) for i in range(50)])
    dst = FlatIndex(dim=d)
    want: list = []

    def check():
        assert len(dst) == len(want)
        for r, (eid, p) in enumerate(want):
            assert dst.id_at(r) == eid and dst.payload_at(r) == p, r
            assert dst.payload(eid) == p

    dst.append_rows_from(src, [3, 7, 9, 11], ["a3", "a7", "a9", "a11"])
    want += [("a3", ("src", 3)), ("a7", ("src", 7)), ("a9", ("src", 9)), ("a11", ("src", 11))]
    check()
    dst.truncate(2)  # cuts into the segment
    del want[2:]
    dst.extend_arrays(["e0"], X[:1], payloads=["explicit"])
    want.append(("e0", "explicit"))
    dst.append_rows_from(src, [20, 21], ["a20", "a21"])
    want += [("a20", ("src", 20)), ("a21", ("src", 21))]
    check()
    dst.insert("a20", X[5], "upserted")  # overwrite a deferred row in place
    want[want.index(("a20", ("src", 20)))] = ("a20", "upserted")
    check()
    dst.clear()
    want.clear()
    dst.append_rows_from(src, [1], ["b1"])
    want.append(("b1", ("src", 1)))
    check()
    assert dst.epoch == 2  # one truncate + one clear


def test_akm_payload_outlives_knowledge_base_changes(gpu):
    """AKM rows settled device-to-device keep deferred payloads (references to
    KB rows).  The reference AKM keeps the Passage object it settled (knowledge.py:217-228),
    so a later upsert, truncation or clear of the KB must not change what the AKM returns."""
    from paper_2506_21593_b200 import AdaptiveKnowledgeMemory, HashEmbedder, Passage, ingest_corpus

    emb = HashEmbedder()
    lines = [json.dumps({"id": f"p{i}", "text": f"passage number {i} about subject {i % 5}", "source": "t"})
             for i in range(40)]
    kb = ingest_corpus(lines, emb)
    akm = AdaptiveKnowledgeMemory()
    akm.settle_from_rows(kb.index, np.array([3, 7, 11, 30], dtype=np.int64))
    before = {pid: akm.index.payload(pid) for pid in ("p3", "p7", "p11", "p30")}
    # upsert p7 in the KB: same id, new passage
    t = "a completely different passage"
    kb.add(Passage(id="p7", text=t, source="t2", embedding=emb.embed(t)))
    assert kb.get("p7").text == t
    assert akm.index.payload("p7") is before["p7"] and akm.index.payload("p7").text != t
    # settle more rows after the upsert: they reference the KB as it is now
    akm.settle_from_rows(kb.index, np.array([7, 12], dtype=np.int64))
    assert akm.index.payload("p12").id == "p12"
    # truncate / clear the KB: settled payloads survive
    kb.index.truncate(20)
    assert akm.index.payload("p30") is before["p30"]
    kb.index.clear()
    assert akm.index.payload("p3") is before["p3"] and akm.index.payload("p12").id == "p12"
