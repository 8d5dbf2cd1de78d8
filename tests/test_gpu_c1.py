"""C1 (BASELINE configs[0]) end to end on the GPU: the reference's nine-session cache-warming
simulation — 100k document chunks, 10k-question pool, dim 384, SimulationConfig(9, 1000,
seed=0) — routed through this package's ``route_batch`` over GPU stores must write session
logs BYTE-IDENTICAL to the ones the real reference's ``run_simulation`` wrote
(simulation.py:268-314; fixture tests/golden/c1_sessions.json.gz from make_c1.py)."""
from __future__ import annotations

import gzip
import json
import os

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def c1():
    with gzip.open(os.path.join(HERE, "golden", "c1_sessions.json.gz"), "rt") as fh:
        return json.load(fh)


@pytest.mark.parametrize("batch", [4096, 256])
def test_c1_route_batch_logs_byte_identical(gpu, c1, batch):
    from benchlib.workloads import corpus_of, qa_rows, simulate_batched
    from paper_2506_21593_b200 import CascadeRouter, HashEmbedder, StubBackend, ingest_corpus

    cfg = c1["config"]
    rows = qa_rows(cfg["kb_rows"], seed=cfg["dataset_seed"])
    emb = HashEmbedder(dim=cfg["dim"])
    kb = ingest_corpus((json.dumps(c) for c in corpus_of(rows)), emb)
    router = CascadeRouter(embedder=emb, backend=StubBackend(), knowledge_base=kb)
    questions = [r["question"] for r in rows[:cfg["qa_rows"]]]
    logs = simulate_batched(router, questions, n_sessions=cfg["n_sessions"], n_queries=cfg["queries_per_session"],
                            seed=cfg["seed"], batch=batch)
    for s, (got, want) in enumerate(zip(logs, c1["sessions"])):
        assert len(got) == len(want)
        bad = [i for i, (a, b) in enumerate(zip(got, want)) if a != b]
        assert not bad, (s, bad[:3], got[bad[0]], want[bad[0]])
    st = router.stats()
    assert {k: v for k, v in st["layer_counts"].items()} == c1["layer_counts"]
