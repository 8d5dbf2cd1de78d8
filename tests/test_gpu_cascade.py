"""route_batch == [route(q) for q in queries], against the reference's recorded runs.

Sequential equivalence is checked three ways: the reference's router trace
(tests/golden/router_trace.json, incl. an AKM hit that forces a batch split),
the reference's two-session simulation logs (tests/golden/simulation.json),
and random replays routed both ways on twin GPU routers under permuted /
disabled layers and a non-empty recall table.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _golden(name):
    with open(os.path.join(HERE, "golden", name)) as fh:
        return json.load(fh)


def _router(corpus, **kw):
    from paper_2506_21593_b200 import CascadeRouter, HashEmbedder, StubBackend, ingest_corpus

    emb = HashEmbedder()
    kb = ingest_corpus((json.dumps(c) for c in corpus), emb)
    backend = kw.pop("backend", None) or StubBackend()
    return CascadeRouter(embedder=emb, backend=backend, knowledge_base=kb, **kw)


def _sig(ans, ev):
    return ([[p.layer.wire_name, p.outcome] for p in ev.layers_probed], ev.serving_layer.wire_name, ans.text,
            list(ans.supporting_passage_ids), [pid for pid, _ in ev.supporting_passages])


@pytest.mark.parametrize("batch,pipelined", [(1000, False), (64, False), (7, False), (64, True), (7, True)])
def test_route_batch_matches_reference_trace(gpu, batch, pipelined):
    """pipelined: ONE route_batch call over the whole trace cut into spans of `batch`, so
    span i+1's device stage runs before span i's host stage (incl. an AKM hit that stops a
    span and discards the speculative next one)."""
    from paper_2506_21593_b200 import validate_query

    gold = _golden("router_trace.json")
    router = _router(gold["corpus"])
    qs = [validate_query(q["text"], "s1", query_id=f"q{i}", issued_at_ns=i) for i, q in enumerate(gold["queries"])]
    got = []
    if pipelined:
        got = router.route_batch(qs, span=batch)
        assert router.last_batch_stats["pipelined"] > 0
    else:
        for i in range(0, len(qs), batch):
            got.extend(router.route_batch(qs[i:i + batch]))
    assert len(got) == len(qs)
    for i, ((ans, ev), q) in enumerate(zip(got, gold["queries"])):
        assert [[p.layer.wire_name, p.outcome] for p in ev.layers_probed] == q["probes"], i
        assert ev.serving_layer.wire_name == q["serving"], i
        assert ans.text == q["answer"], i
        assert list(ans.supporting_passage_ids) == q["passages"], i
    st, g = router.stats(), gold["stats"]
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


def test_route_batch_matches_reference_simulation(gpu):
    from paper_2506_21593_b200 import validate_query

    gold = _golden("simulation.json")
    router = _router(gold["corpus"])
    for lines in gold["sessions"]:
        recs = [json.loads(ln) for ln in lines]
        router.reset_session()
        qs = [validate_query(r["query_text"], r["session_id"], query_id=r["query_id"], issued_at_ns=r["timestamp_ns"])
              for r in recs]
        got = router.route_batch(qs)
        for i, ((ans, ev), r) in enumerate(zip(got, recs)):
            assert [[p.layer.wire_name, p.outcome] for p in ev.layers_probed] == \
                [[p["layer"], p["outcome"]] for p in r["layers_probed"]], i
            assert ev.serving_layer.wire_name == r["serving_layer"], i
            assert ans.text == r["answer_text"], i
            assert [pid for pid, _ in ev.supporting_passages] == [p["id"] for p in r["supporting_passages"]], i


@pytest.mark.parametrize("one_call", [True, False], ids=["pr_cascade_route", "python_orchestration"])
@pytest.mark.parametrize("span", [4096, 29])
@pytest.mark.parametrize("variant", ["default", "permuted", "disabled", "recall", "device_recall",
                                     "device_recall_first"])
def test_route_batch_equals_sequential_random(gpu, variant, span, one_call, monkeypatch):
    """Both device-stage orchestrations of a span (the one-call pr_cascade_route and the
    same calls issued one by one from Python) against sequential route().
    device_recall*: the batched router's recall table is a DeviceKnowledgeTable (L3
    decided on the device, pr_recall_gate), the sequential twin's the host
    StubKnowledgeTable with the same adds — low confidences, empty answers, overwrites,
    an inclusive threshold boundary, and L3 probed first."""
    from paper_2506_21593_b200 import (DeviceKnowledgeTable, LayerTag, RouterConfig, StubBackend, StubKnowledgeTable,
                                       cascade, validate_query)

    monkeypatch.setattr(cascade, "_ROUTE_C", one_call)
    gold = _golden("simulation.json")
    corpus, questions = gold["corpus"][:150], gold["questions"]
    kw = {}
    if variant == "permuted":
        kw["config"] = RouterConfig(layer_order=(LayerTag.SEMANTIC_CACHE, LayerTag.ADAPTIVE_MEMORY,
                                                 LayerTag.FIXED_KV, LayerTag.MEMORY_RECALL, LayerTag.NAIVE_RAG))
    elif variant == "disabled":
        kw["config"] = RouterConfig(disabled_layers=frozenset({LayerTag.FIXED_KV, LayerTag.MEMORY_RECALL}))
    elif variant == "device_recall_first":
        kw["config"] = RouterConfig(layer_order=(LayerTag.MEMORY_RECALL, LayerTag.FIXED_KV, LayerTag.SEMANTIC_CACHE,
                                                 LayerTag.ADAPTIVE_MEMORY, LayerTag.NAIVE_RAG), recall_threshold=0.3)
    rng = np.random.default_rng(5)
    texts = []
    for i in range(300):
        if texts and rng.random() < 0.5:
            t = texts[int(rng.integers(len(texts)))]
            if rng.random() < 0.5:
                t = t.rstrip("?") if t.endswith("?") else t + "?"
        else:
            t = questions[int(rng.integers(len(questions)))]
        texts.append(t)
    # passages that equal later queries make AKM hits (and batch splits) likely
    texts[150:150] = [corpus[3]["text"], corpus[7]["text"]]

    def mk(device=False):
        extra = dict(kw)
        if variant == "recall":
            tab = StubKnowledgeTable()
            for t in texts[::9]:
                tab.add(t, "recalled " + t[:10], 0.9)
            extra["backend"] = StubBackend(tab)
        elif variant.startswith("device_recall"):
            tab = DeviceKnowledgeTable() if device else StubKnowledgeTable()
            for t in texts[::9]:
                tab.add(t, "recalled " + t[:10], 0.9)
            for t in texts[2::11]:
                tab.add(t, "shaky " + t[:8], 0.3)  # rejected at 0.5, accepted at 0.3 (inclusive)
            for t in texts[4::13]:
                tab.add(t, "", 0.95)  # an empty answer is never accepted
            for t in texts[::27]:
                tab.add(t, "rewritten " + t[:6], 0.6)  # overwrite: the latest add wins
            extra["backend"] = StubBackend(tab)
        return _router(corpus, **extra)

    seq, bat = mk(), mk(device=True)
    qs = [validate_query(t, "s", query_id=f"q{i}", issued_at_ns=i) for i, t in enumerate(texts)]
    want = [_sig(*seq.route(q)) for q in qs]
    got = []
    for i in range(0, len(qs), 97):
        got.extend(_sig(*r) for r in bat.route_batch(qs[i:i + 97], span=span))
    assert got == want
    assert seq.stats() == bat.stats()
    assert seq.backend.context_calls == bat.backend.context_calls
    assert seq.backend.recall_calls == bat.backend.recall_calls
    assert seq.adaptive_memory.ids() == bat.adaptive_memory.ids()
    assert seq.adaptive_memory.index.entry_ids() == bat.adaptive_memory.index.entry_ids()
    assert seq.adaptive_memory.pending_count() == bat.adaptive_memory.pending_count()
    assert seq.semantic_cache.index.entry_ids() == bat.semantic_cache.index.entry_ids()
    assert seq.semantic_cache.index.search_count == bat.semantic_cache.index.search_count
    assert seq.adaptive_memory.index.search_count == bat.adaptive_memory.index.search_count
    assert seq.knowledge_base.index.search_count == bat.knowledge_base.index.search_count
    assert [e["query_text"] for e in seq.kv_cache.export_entries()] == \
        [e["query_text"] for e in bat.kv_cache.export_entries()]


def test_batched_simulation_logs_byte_identical(gpu):
    """f3: session logs materialised from batched routing are byte-identical to
    the reference's run_simulation output (simulation.py:268-314)."""
    from benchlib.workloads import simulate_batched

    gold = _golden("simulation.json")
    router = _router(gold["corpus"])
    logs = simulate_batched(router, gold["questions"], n_sessions=gold["n_sessions"],
                            n_queries=gold["queries_per_session"], seed=gold["seed"], batch=64)
    for s, (got, want) in enumerate(zip(logs, gold["sessions"])):
        for i, (a, b) in enumerate(zip(got, want)):
            assert a == b, (s, i)
        assert len(got) == len(want)


def test_concurrent_sessions_share_knowledge_base(gpu):
    """Two routers (own caches / AKM) over ONE knowledge base, routing their sessions
    from two threads at once (the C5 bench's session workers): each gets exactly what
    it gets routing alone, and the shared KB's search counter sums both."""
    import threading

    from paper_2506_21593_b200 import CascadeRouter, HashEmbedder, StubBackend, ingest_corpus, validate_query

    gold = _golden("simulation.json")
    emb = HashEmbedder()
    kb = ingest_corpus((json.dumps(c) for c in gold["corpus"]), emb)
    rng = np.random.default_rng(9)
    sessions = []
    for s in range(2):
        texts = []
        for i in range(400):
            if texts and rng.random() < 0.5:
                texts.append(texts[int(rng.integers(len(texts)))])
            else:
                texts.append(gold["questions"][int(rng.integers(len(gold["questions"])))])
        sessions.append([validate_query(t, f"s{s}", query_id=f"s{s}q{i}", issued_at_ns=i)
                         for i, t in enumerate(texts)])

    def mk():
        return CascadeRouter(embedder=emb, backend=StubBackend(), knowledge_base=kb)

    def run(router, qs, out):
        for i in range(0, len(qs), 64):
            out.extend(_sig(*r) for r in router.route_batch(qs[i:i + 64]))

    c0 = kb.index.search_count
    alone = []
    for qs in sessions:
        out: list = []
        run(mk(), qs, out)
        alone.append(out)
    c1 = kb.index.search_count
    routers, outs = [mk(), mk()], [[], []]
    threads = [threading.Thread(target=run, args=(routers[s], sessions[s], outs[s])) for s in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert outs == alone
    assert kb.index.search_count - c1 == c1 - c0  # the shared counter saw every probe of both


def test_route_batch_backend_failure_rolls_back(gpu):
    """A backend that raises mid-batch (BackendUnavailable from a remote LLM,
    generation.py:118-175) must leave the stores as independent route() calls would:
    the batch's pre-appended semantic-cache rows are rolled back, the span is re-routed
    query by query, and with capture_errors only the failing query gets the error."""
    from paper_2506_21593_b200 import BackendUnavailable, StubBackend, validate_query

    class Flaky(StubBackend):
        def generate_with_context(self, query_text, passages):
            if query_text.startswith("BOOM"):
                self.context_calls += 1
                raise BackendUnavailable("remote backend down")
            return super().generate_with_context(query_text, passages)

    gold = _golden("simulation.json")
    corpus, questions = gold["corpus"][:150], gold["questions"]
    texts = [questions[i % 40] for i in range(120)]
    texts[50] = "BOOM " + questions[77]
    texts[90] = texts[50]  # the failed query is not cached: it fails again
    seq, bat = _router(corpus, backend=Flaky()), _router(corpus, backend=Flaky())
    qs = [validate_query(t, "s", query_id=f"q{i}", issued_at_ns=i) for i, t in enumerate(texts)]

    def sig(r):
        return ("error", type(r).__name__) if isinstance(r, Exception) else _sig(*r)

    want = []
    for q in qs:
        try:
            want.append(sig(seq.route(q)))
        except BackendUnavailable as exc:
            want.append(sig(exc))
    got = []
    for i in range(0, len(qs), 64):
        got.extend(sig(r) for r in bat.route_batch(qs[i:i + 64], capture_errors=True, span=16))
    assert got == want
    assert got[50] == ("error", "BackendUnavailable")
    assert seq.stats() == bat.stats()
    assert seq.backend.context_calls == bat.backend.context_calls
    assert seq.semantic_cache.index.entry_ids() == bat.semantic_cache.index.entry_ids()
    assert all(p is not None for p in bat.semantic_cache.index._payloads)
    with pytest.raises(BackendUnavailable):
        bat.route_batch([validate_query(texts[50], "s", query_id="x", issued_at_ns=0)])
