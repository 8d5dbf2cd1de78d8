"""The drop-in, end to end: the REAL reference router (``ragcascade.CascadeRouter``,
installed offline into baseline/_ref — git-ignored, it travels to the GPU box with the
tree) driving this package's GPU stores through the injection surface
(src/router.py:195-223), replaying the reference's recorded 201-query trace.  Skipped
when the reference install is absent; nothing reads /root/reference at run time."""
from __future__ import annotations

import json
import os
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(os.path.dirname(HERE), "baseline", "_ref")


@pytest.fixture(scope="module")
def rc():
    if not os.path.isdir(os.path.join(REF, "ragcascade")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import ragcascade
    finally:
        sys.path.remove(REF)
    return ragcascade


def test_reference_router_over_gpu_stores_replays_trace(gpu, rc):
    import paper_2506_21593_b200 as g

    with open(os.path.join(HERE, "golden", "router_trace.json")) as fh:
        gold = json.load(fh)
    emb = rc.HashEmbedder()
    kb = g.ingest_corpus((json.dumps(c) for c in gold["corpus"]), emb)  # GPU store, reference vectors
    router = rc.CascadeRouter(
        embedder=emb, backend=rc.StubBackend(), knowledge_base=kb,
        kv_cache=g.FixedKVCache(), semantic_cache=g.SemanticCache(emb), adaptive_memory=g.AdaptiveKnowledgeMemory(),
    )
    for i, q in enumerate(gold["queries"]):
        if q["origin"] == "akm_probe":
            router.adaptive_memory.settle()
        answer, ev = router.route(rc.validate_query(q["text"], "s1"))
        assert [[p.layer.wire_name, p.outcome] for p in ev.layers_probed] == q["probes"], i
        assert ev.serving_layer.wire_name == q["serving"], i
        assert answer.text == q["answer"], i
        assert list(answer.supporting_passage_ids) == q["passages"], i
    st, want = router.stats(), gold["stats"]
    assert st["layer_counts"] == want["layer_counts"]
    assert router.semantic_cache.index.search_count == want["sc_searches"]
    assert router.adaptive_memory.index.search_count == want["akm_searches"]
    assert router.adaptive_memory.inserted_total == want["akm_inserted_total"]


def test_reference_simulation_over_gpu_stores_logs_identical(gpu, rc):
    """The reference's own simulation driver (run_simulation, two sessions) over the reference
    router with every store replaced by its GPU drop-in writes session logs byte-identical to
    the ones the reference wrote with its own stores (tests/golden/simulation.json)."""
    import paper_2506_21593_b200 as g
    from ragcascade.datagen import synthetic_qa_dataset
    from ragcascade.simulation import dataset_to_corpus

    with open(os.path.join(HERE, "golden", "simulation.json")) as fh:
        gold = json.load(fh)
    emb = rc.HashEmbedder()
    rows = synthetic_qa_dataset(gold["dataset_n"], seed=42)
    kb = g.ingest_corpus((json.dumps(r) for r in dataset_to_corpus(rows)), emb)
    router = rc.CascadeRouter(
        embedder=emb, backend=rc.StubBackend(), knowledge_base=kb,
        kv_cache=g.FixedKVCache(), semantic_cache=g.SemanticCache(emb), adaptive_memory=g.AdaptiveKnowledgeMemory(),
    )
    cfg = rc.SimulationConfig(n_sessions=gold["n_sessions"], queries_per_session=gold["queries_per_session"],
                              seed=gold["seed"])
    logs = rc.run_simulation(cfg, router, rows)
    assert [list(log.to_jsonl_lines()) for log in logs] == gold["sessions"]


def test_reference_stores_on_gpu_flatindex_logs_identical(gpu, rc, monkeypatch):
    """Module-level substitution: the reference's OWN caches, AKM and
    knowledge base, with ``FlatIndex`` re-bound to the GPU index in their modules, run the
    reference simulation to byte-identical session logs."""
    import ragcascade.caches as rcc
    import ragcascade.index as rci
    import ragcascade.knowledge as rck
    from ragcascade.datagen import synthetic_qa_dataset
    from ragcascade.simulation import dataset_to_corpus

    from paper_2506_21593_b200 import FlatIndex as GpuFlatIndex

    for mod in (rc, rci, rcc, rck):
        if hasattr(mod, "FlatIndex"):
            monkeypatch.setattr(mod, "FlatIndex", GpuFlatIndex)
    with open(os.path.join(HERE, "golden", "simulation.json")) as fh:
        gold = json.load(fh)
    emb = rc.HashEmbedder()
    rows = synthetic_qa_dataset(gold["dataset_n"], seed=42)
    kb = rc.MainKnowledgeBase()
    rc.ingest_corpus((json.dumps(r) for r in dataset_to_corpus(rows)), emb, kb=kb)
    assert isinstance(kb.index, GpuFlatIndex)
    router = rc.CascadeRouter(embedder=emb, backend=rc.StubBackend(), knowledge_base=kb)
    assert isinstance(router.semantic_cache.index, GpuFlatIndex)
    cfg = rc.SimulationConfig(n_sessions=gold["n_sessions"], queries_per_session=gold["queries_per_session"],
                              seed=gold["seed"])
    logs = rc.run_simulation(cfg, router, rows)
    assert [list(log.to_jsonl_lines()) for log in logs] == gold["sessions"]
