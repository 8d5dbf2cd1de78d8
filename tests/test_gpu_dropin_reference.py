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
    stores = dict(kv_cache=g.FixedKVCache(), semantic_cache=g.SemanticCache(emb),
                  adaptive_memory=g.AdaptiveKnowledgeMemory())
    router = rc.CascadeRouter(embedder=emb, backend=rc.StubBackend(), knowledge_base=kb, **stores)
    for name, store in stores.items():  # empty drop-ins are truthy: the router keeps them (router.py:213-220)
        assert getattr(router, name) is store
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
    stores = dict(kv_cache=g.FixedKVCache(), semantic_cache=g.SemanticCache(emb),
                  adaptive_memory=g.AdaptiveKnowledgeMemory())
    router = rc.CascadeRouter(embedder=emb, backend=rc.StubBackend(), knowledge_base=kb, **stores)
    for name, store in stores.items():  # empty drop-ins are truthy: the router keeps them (router.py:213-220)
        assert getattr(router, name) is store
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


def _sim_logs(rc, router, rows, n_sessions=2, per_session=150, seed=23):
    cfg = rc.SimulationConfig(n_sessions=n_sessions, queries_per_session=per_session, seed=seed)
    return [list(log.to_jsonl_lines()) for log in rc.run_simulation(cfg, router, rows)]


@pytest.mark.parametrize("variant", ["lru_caches", "permuted", "disabled", "recall_table", "thresholds",
                                     "device_recall_table"])
def test_live_ab_against_reference_stores(gpu, rc, variant):
    """Live A/B on the GPU box: the reference simulation through the reference router, once
    with the reference's own stores and once with the GPU drop-ins (same config, same seed),
    under capped caches (LRU / recency eviction), permuted and disabled layers, a recall
    table, and non-default thresholds.  Session logs must be byte-identical."""
    import paper_2506_21593_b200 as g
    from ragcascade.datagen import synthetic_qa_dataset
    from ragcascade.simulation import dataset_to_corpus

    L = rc.LayerTag
    rows = synthetic_qa_dataset(300, seed=42)
    corpus = [json.dumps(r) for r in dataset_to_corpus(rows)]
    emb = rc.HashEmbedder()
    cfg_kw, kv_kw, sc_kw = {}, {}, {}
    if variant == "lru_caches":
        kv_kw, sc_kw = {"max_entries": 40}, {"max_entries": 30}
    elif variant == "permuted":
        cfg_kw["layer_order"] = (L.SEMANTIC_CACHE, L.ADAPTIVE_MEMORY, L.FIXED_KV, L.MEMORY_RECALL, L.NAIVE_RAG)
    elif variant == "disabled":
        cfg_kw["disabled_layers"] = frozenset({L.FIXED_KV, L.ADAPTIVE_MEMORY})
    elif variant == "thresholds":
        cfg_kw.update(semantic_threshold=0.6, akm_threshold=0.5, retrieval_k=2, akm_seed_k=5)

    def backend(stores):
        # device_recall_table: the reference's StubBackend over the GPU recall table
        tab = g.DeviceKnowledgeTable() if variant == "device_recall_table" and stores == "gpu" else \
            rc.StubKnowledgeTable()
        if variant in ("recall_table", "device_recall_table"):
            for i, r in enumerate(rows[::5]):
                tab.add(r["question"], "recalled: " + r["answer"], 0.8 if i % 4 else 0.4)
        return rc.StubBackend(tab)

    def build(stores):
        cfg = rc.RouterConfig(**cfg_kw)
        if stores == "ref":
            kb = rc.MainKnowledgeBase()
            rc.ingest_corpus(iter(corpus), emb, kb=kb)
            kw = dict(kv_cache=rc.FixedKVCache(**kv_kw),
                      semantic_cache=rc.SemanticCache(emb, threshold=cfg.semantic_threshold, **sc_kw),
                      adaptive_memory=rc.AdaptiveKnowledgeMemory(threshold=cfg.akm_threshold))
        else:
            kb = g.ingest_corpus(iter(corpus), emb)
            kw = dict(kv_cache=g.FixedKVCache(**kv_kw),
                      semantic_cache=g.SemanticCache(emb, threshold=cfg.semantic_threshold, **sc_kw),
                      adaptive_memory=g.AdaptiveKnowledgeMemory(threshold=cfg.akm_threshold))
        r = rc.CascadeRouter(embedder=emb, backend=backend(stores), knowledge_base=kb, config=cfg, **kw)
        # the reference injects with ``kv_cache or FixedKVCache()`` (router.py:213-220): its OWN
        # empty stores are falsy and get replaced (dropping e.g. max_entries); pin the stores
        # passed on both sides so the A/B compares exactly these stores
        for name, store in kw.items():
            setattr(r, name, store)
        return r

    want = _sim_logs(rc, build("ref"), rows)
    got = _sim_logs(rc, build("gpu"), rows)
    assert got == want


@pytest.mark.parametrize("variant", ["default", "permuted", "disabled", "recall_table", "thresholds",
                                     "device_recall_table", "device_recall_first"])
def test_live_ab_route_batch_against_reference(gpu, rc, variant):
    """This package's CascadeRouter.route_batch (batches of 64, GPU stores) against the
    reference's run_simulation with the reference router and stores, live on the box:
    session logs byte-identical under each router configuration."""
    import paper_2506_21593_b200 as g
    from benchlib.workloads import simulate_batched
    from ragcascade.datagen import synthetic_qa_dataset
    from ragcascade.simulation import dataset_to_corpus

    rows = synthetic_qa_dataset(300, seed=42)
    corpus = [json.dumps(r) for r in dataset_to_corpus(rows)]

    def cfg_kw(L):
        if variant == "permuted":
            return {"layer_order": (L.SEMANTIC_CACHE, L.ADAPTIVE_MEMORY, L.FIXED_KV, L.MEMORY_RECALL, L.NAIVE_RAG)}
        if variant == "disabled":
            return {"disabled_layers": frozenset({L.FIXED_KV, L.MEMORY_RECALL})}
        if variant == "thresholds":
            return {"semantic_threshold": 0.6, "akm_threshold": 0.5, "retrieval_k": 2, "akm_seed_k": 5}
        if variant == "device_recall_first":
            return {"layer_order": (L.MEMORY_RECALL, L.FIXED_KV, L.SEMANTIC_CACHE, L.ADAPTIVE_MEMORY, L.NAIVE_RAG),
                    "recall_threshold": 0.4}
        return {}

    def table(mod):
        # device_recall_*: this package's side keeps the table on the GPU (L3 decided by
        # pr_recall_gate inside route_batch); the reference keeps its dict
        dev = variant.startswith("device_recall") and mod is g
        tab = g.DeviceKnowledgeTable() if dev else mod.StubKnowledgeTable()
        if variant == "recall_table" or variant.startswith("device_recall"):
            for i, r in enumerate(rows[::5]):
                tab.add(r["question"], "recalled: " + r["answer"], 0.8 if i % 4 else 0.4)
            if variant.startswith("device_recall"):
                for r in rows[1::17]:
                    tab.add(r["question"], "", 0.9)  # empty answers are rejected
        return tab

    # reference: its own router, stores and simulation driver
    emb_r = rc.HashEmbedder()
    kb_r = rc.MainKnowledgeBase()
    rc.ingest_corpus(iter(corpus), emb_r, kb=kb_r)
    cfg_r = rc.RouterConfig(**cfg_kw(rc.LayerTag))
    ref = rc.CascadeRouter(embedder=emb_r, backend=rc.StubBackend(table(rc)), knowledge_base=kb_r, config=cfg_r,
                           semantic_cache=rc.SemanticCache(emb_r, threshold=cfg_r.semantic_threshold),
                           adaptive_memory=rc.AdaptiveKnowledgeMemory(threshold=cfg_r.akm_threshold))
    sim = rc.SimulationConfig(n_sessions=2, queries_per_session=150, seed=29)
    want = [list(log.to_jsonl_lines()) for log in rc.run_simulation(sim, ref, rows)]
    # this package: route_batch over the GPU stores
    emb = g.HashEmbedder()
    cfg = g.RouterConfig(**cfg_kw(g.LayerTag))
    mine = g.CascadeRouter(embedder=emb, backend=g.StubBackend(table(g)), knowledge_base=g.ingest_corpus(iter(corpus), emb),
                           config=cfg, semantic_cache=g.SemanticCache(emb, threshold=cfg.semantic_threshold),
                           adaptive_memory=g.AdaptiveKnowledgeMemory(threshold=cfg.akm_threshold))
    got = simulate_batched(mine, [r["question"] for r in rows], n_sessions=2, n_queries=150, seed=29, batch=64)
    assert got == want


@pytest.mark.parametrize("mode_name", ["MODE_EXACT", "MODE_TENSOR", "MODE_TENSOR_I8", "MODE_AUTO"])
def test_live_flatindex_search_against_reference(gpu, rc, rng, mode_name):
    """GPU FlatIndex.search against the reference's own FlatIndex.search, live: ids, ranks
    and score bits, on a store with exact duplicates (tie tiers), self-hits and near-hits."""
    import numpy as np

    import paper_2506_21593_b200 as g
    from conftest import random_unit_vectors

    mode = getattr(g, mode_name)
    n, d = 6000, 256
    X = random_unit_vectors(rng, n, d)
    X[100:140] = X[7]  # a tier of 41 bit-identical rows
    ref, mine = rc.FlatIndex(dim=d), g.FlatIndex(dim=d)
    ids = [f"e{i}" for i in range(n)]
    for i in range(n):
        ref.insert(ids[i], X[i])
    mine.extend_arrays(ids, X)
    Q = random_unit_vectors(rng, 40, d)
    Q[0], Q[1] = X[7], X[2500]  # self-hits (snap) incl. the tied tier
    for i in range(2, 12):
        v = X[int(rng.integers(n))] + 0.02 * random_unit_vectors(rng, 1, d)[0]
        Q[i] = (v / np.linalg.norm(v.astype(np.float64))).astype(np.float32)
    for k in (1, 5, 10):
        for q in Q:
            want = ref.search(q, k)
            got = mine.search(q, k, mode=mode)
            assert [(h.entry_id, h.score, h.rank) for h in got] == [(h.entry_id, h.score, h.rank) for h in want]


def test_live_snapshot_interop_with_reference(gpu, rc, rng):
    """RCFLATIX both ways, live: the reference restores the GPU index's snapshot and the GPU
    index restores the reference's, each searching to the same hits."""
    import paper_2506_21593_b200 as g
    from conftest import random_unit_vectors

    d = 64
    X = random_unit_vectors(rng, 500, d)
    ref = rc.FlatIndex(dim=d)
    for i in range(500):
        ref.insert(f"r{i}", X[i], {"i": i})
    ref.insert("r3", X[9], {"i": "upserted"})
    mine = g.FlatIndex.restore(ref.snapshot())
    back = rc.FlatIndex.restore(mine.snapshot())
    assert mine.snapshot() == ref.snapshot() == back.snapshot()
    for q in random_unit_vectors(rng, 10, d):
        want = [(h.entry_id, h.score) for h in ref.search(q, 7)]
        assert [(h.entry_id, h.score) for h in mine.search(q, 7)] == want
        assert [(h.entry_id, h.score) for h in back.search(q, 7)] == want


def test_live_hash_embedder_against_reference(gpu, rc):
    """Device HashEmbedder against the reference's HashEmbedder on mixed texts (ASCII, unicode
    word characters, punctuation-only, long), bit for bit."""
    import numpy as np

    import paper_2506_21593_b200 as g

    texts = ["What is the capital of France?", "naïve café über straße", "日本語のテキスト", "!!! ??? ...",
             "x", "a_b c-d e.f", " ".join(f"tok{i}" for i in range(300)), "Mixed 123 numbers 4.5e6",
             "tab\tseparated\nlines", "emoji 🙂 inside"]
    texts += [f"question {i} about topic {i % 13} and item {i * 7}" for i in range(500)]
    ref, mine = rc.HashEmbedder(), g.HashEmbedder()
    V = mine.embed_device(texts).cpu().numpy()
    for t, v in zip(texts, V):
        w = np.asarray(ref.embed(t).values, dtype=np.float32)
        assert np.array_equal(v, w), t


@pytest.mark.parametrize("max_entries", [None, 25])
def test_live_kv_cache_random_ops_against_reference(gpu, rc, rng, max_entries):
    """Random put / get / clear sequences on the reference FixedKVCache and the GPU table
    (unbounded and LRU-capped): every get, hit/miss counter and size agrees."""
    import paper_2506_21593_b200 as g

    ref, mine = rc.FixedKVCache(max_entries=max_entries), g.FixedKVCache(max_entries=max_entries)
    keys = [f"key {i}" for i in range(60)] + ["", "é", "key 1 ", "KEY 1"]
    for step in range(1500):
        op = rng.random()
        t = keys[int(rng.integers(len(keys)))]
        if op < 0.45:
            a = rc.AnswerRecord(text=f"answer {step}", layer=rc.LayerTag.NAIVE_RAG, confidence=0.5,
                                supporting_passage_ids=("p",))
            ref.put(t, a)
            mine.put(t, a)
        elif op < 0.995:
            x, y = ref.get(t), mine.get(t)
            assert (x is None) == (y is None), step
            if x is not None:
                assert (x.text, x.layer.wire_name) == (y.text, y.layer.wire_name), step
        else:
            ref.clear()
            mine.clear()
        assert len(ref) == len(mine), step
    assert (ref.hits, ref.misses) == (mine.hits, mine.misses)
