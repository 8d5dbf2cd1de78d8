"""L3 memory recall on the device: ``DeviceKnowledgeTable`` is the
reference's ``StubKnowledgeTable`` (src/generation.py:51-80) kept in a fixed-KV device
table, and ``pr_recall_gate`` is ``memory_recall``'s confidence gate
(src/generation.py:203-224) for a whole routed span."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_table_matches_host_table(gpu):
    """add / overwrite / lookup / len / bad confidence, against the host restatement
    (itself the reference's dict semantics)."""
    from paper_2506_21593_b200 import DeviceKnowledgeTable, StubKnowledgeTable

    rng = np.random.default_rng(3)
    dev, host = DeviceKnowledgeTable(capacity=64), StubKnowledgeTable()
    assert len(dev) == 0 and bool(dev)  # an empty table stays the table (generation.py:95)
    keys = [f"Question {i}?" for i in range(500)] + ["", "é unicode ✓", "x" * 300, "Question 1? "]
    for _ in range(3000):
        k = keys[int(rng.integers(len(keys)))]
        a = "" if rng.random() < 0.1 else f"answer {int(rng.integers(1 << 30))}"
        c = float(rng.choice([0.0, 0.3, 0.5, 0.9, 1.0]))
        dev.add(k, a, c)
        host.add(k, a, c)
    assert len(dev) == len(host)
    for k in keys + ["never added", "question 1?"]:
        assert dev.lookup(k) == host.lookup(k), k
    for bad in (-0.1, 1.5, float("nan")):
        with pytest.raises(ValueError):
            dev.add("q", "a", bad)
    with pytest.raises(ValueError):
        dev.add_many(["a", "b"], ["x", "y"], [0.5, 2.0])  # validated before anything is inserted
    assert dev.lookup("a") is None


def test_gate_device_equals_memory_recall(gpu):
    """pr_recall_gate over a batch == memory_recall per query at several thresholds
    (inclusive boundary, empty answers never accepted)."""
    from paper_2506_21593_b200 import DeviceKnowledgeTable, StubBackend, StubKnowledgeTable, memory_recall
    from paper_2506_21593_b200 import validate_query
    from paper_2506_21593_b200.textarena import to_device

    dev, host = DeviceKnowledgeTable(), StubKnowledgeTable()
    qs = [f"q{i}" for i in range(1000)]
    for i, q in enumerate(qs[:700]):
        a = "" if i % 10 == 3 else f"a{i}"
        c = [0.0, 0.25, 0.5, 0.75, 1.0][i % 5]
        dev.add(q, a, c)
        host.add(q, a, c)
    arena = to_device(qs)
    for thr in (0.0, 0.25, 0.5, 0.9, 1.0):
        vals, ok = dev.gate_device(arena[0], arena[1], len(qs), thr)
        ok, vals = ok.cpu().numpy().astype(bool), vals.cpu().numpy()
        be = StubBackend(host)
        for j, q in enumerate(qs):
            rec = memory_recall(be, validate_query(q, "s"), thr)
            assert ok[j] == (rec is not None), (thr, q)
            if rec is not None:
                e = dev.entry_at(int(vals[j]))
                assert (e.answer, e.confidence) == (rec.text, rec.confidence)
    with pytest.raises(ValueError):  # memory_recall's ValueError (generation.py:214-215)
        dev.gate_device(arena[0], arena[1], len(qs), 1.5)


def test_from_triples_jsonl(gpu, tmp_path):
    from paper_2506_21593_b200 import DeviceKnowledgeTable, MalformedJsonl, StubKnowledgeTable

    p = tmp_path / "t.jsonl"
    p.write_text('{"question": "Q1?", "context": "c", "answer": "A1"}\n\n{"question": "Q2?", "answer": "A2"}\n'
                 '{"question": "Q1?", "answer": "A1b"}\n', encoding="utf-8")
    dev = DeviceKnowledgeTable.from_triples_jsonl(p, confidence=0.7)
    host = StubKnowledgeTable.from_triples_jsonl(p, confidence=0.7)
    assert len(dev) == len(host) == 2
    for q in ("Q1?", "Q2?", "Q3?"):
        assert dev.lookup(q) == host.lookup(q)
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"question": "Q", "answer": "A"}\n[1, 2]\n', encoding="utf-8")
    with pytest.raises(MalformedJsonl) as ei:
        DeviceKnowledgeTable.from_triples_jsonl(bad)
    assert ei.value.line_number == 2


@pytest.mark.parametrize("batched", [False, True])
def test_knowledge_migration_loop(gpu, batched):
    """The reference's migration acceptance test (pkg/tests/test_acceptance.py:251-271) with
    the recall table on the device: after a session, the exported training triples are
    loaded into a DeviceKnowledgeTable and every triple's question is served by L3 when
    replayed — through route() and through route_batch (L3 decided on the device)."""
    from benchlib.workloads import simulate_batched
    from paper_2506_21593_b200 import (CascadeRouter, DeviceKnowledgeTable, HashEmbedder, LayerTag, StubBackend,
                                       export_triples, ingest_corpus, validate_query)

    with open(os.path.join(HERE, "golden", "simulation.json")) as fh:
        gold = json.load(fh)
    emb = HashEmbedder()
    router = CascadeRouter(embedder=emb, backend=StubBackend(),
                           knowledge_base=ingest_corpus((json.dumps(c) for c in gold["corpus"]), emb))
    simulate_batched(router, gold["questions"], n_sessions=1, n_queries=300, seed=5, batch=64)
    triples = list(export_triples(router.trace.events()))
    assert triples
    table = DeviceKnowledgeTable()
    for t in triples:
        table.add(t.question, t.answer)
    router.backend = StubBackend(knowledge=table)
    router.latency_model = None
    router.reset_session()
    qs = [validate_query(t.question, "replay") for t in triples]
    if batched:
        got = router.route_batch(qs)
        assert router.last_batch_stats["batched"] == len(qs)
    else:
        got = [router.route(q) for q in qs]
    assert all(a.layer is LayerTag.MEMORY_RECALL for a, _ in got)
    assert [a.text for a, _ in got] == [t.answer for t in triples]
    assert router.backend.recall_calls == len(qs)
