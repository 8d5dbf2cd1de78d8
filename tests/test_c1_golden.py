"""C1 (BASELINE configs[0]) golden fixture, CPU side: the reference's nine-session
``run_simulation`` at 100k chunks x dim 384 (tests/golden/c1_sessions.json.gz, written by
tests/golden/make_c1.py from the real reference) is internally consistent, and this repo's
workload generators reproduce its query streams — so the GPU test (test_gpu_c1.py) routes
exactly the reference's queries."""
from __future__ import annotations

import gzip
import hashlib
import json
import os

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def c1():
    with gzip.open(os.path.join(HERE, "golden", "c1_sessions.json.gz"), "rt") as fh:
        return json.load(fh)


def test_c1_fixture_shape_and_digests(c1):
    cfg = c1["config"]
    assert (cfg["kb_rows"], cfg["qa_rows"], cfg["dim"]) == (100_000, 10_000, 384)
    assert (cfg["n_sessions"], cfg["queries_per_session"], cfg["seed"]) == (9, 1000, 0)
    assert len(c1["sessions"]) == 9
    for lines, digest in zip(c1["sessions"], c1["sha256"]):
        assert len(lines) == 1000
        assert hashlib.sha256("\n".join(lines).encode()).hexdigest() == digest
    served = {}
    for lines in c1["sessions"]:
        for ln in lines:
            layer = json.loads(ln)["serving_layer"]
            served[layer] = served.get(layer, 0) + 1
    assert served == {k: v for k, v in c1["layer_counts"].items() if v}
    assert served["naive_rag"] > 4000  # half the C1 stream reaches the 100k-chunk scan


def test_c1_streams_reproduced_by_workload_generators(c1):
    from benchlib.workloads import qa_rows, session_stream

    questions = [r["question"] for r in qa_rows(c1["config"]["qa_rows"], seed=c1["config"]["dataset_seed"])]
    for s, lines in enumerate(c1["sessions"]):
        recs = [json.loads(ln) for ln in lines]
        sid, stream = session_stream(questions, 1000, c1["config"]["seed"], s)
        assert sid == recs[0]["session_id"]
        assert [t for t, _ in stream] == [r["query_text"] for r in recs]
        assert [o for _, o in stream] == [r["origin"] for r in recs]


def test_c1_corpus_matches_reference_datagen(c1):
    """The 100k-row corpus the GPU test ingests equals the reference's dataset_to_corpus of
    synthetic_qa_dataset(100_000, 42) — checked live when the reference is importable."""
    from benchlib.workloads import corpus_of, qa_rows
    from oracle import ref_c1

    try:
        rc = ref_c1.load_reference()
    except ImportError:
        pytest.skip("reference not importable here")
    from ragcascade.simulation import dataset_to_corpus

    ref_rows = ref_c1.c1_rows(rc)
    rows = qa_rows(100_000, seed=42)
    assert rows == ref_rows
    assert corpus_of(rows) == dataset_to_corpus(ref_rows)
