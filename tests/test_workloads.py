"""The workload generators reproduce the reference's recorded streams (CPU only)."""
from __future__ import annotations

import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def _sim():
    with open(os.path.join(HERE, "golden", "simulation.json")) as fh:
        return json.load(fh)


def test_qa_rows_match_reference_dataset():
    from benchlib.workloads import corpus_of, qa_rows

    g = _sim()
    rows = qa_rows(g["dataset_n"], seed=42)
    assert [r["question"] for r in rows] == g["questions"]
    assert corpus_of(rows) == g["corpus"]


def test_vector_latency_draws_equal_scalar_draws():
    import numpy as np

    from benchlib.workloads import LatencyDraws

    a, b = LatencyDraws(0.25, [3, 1, 1]), LatencyDraws(0.25, [3, 1, 1])
    layers = np.random.default_rng(0).integers(1, 6, 500)
    many = a.sample_many(layers)
    one = np.array([b.sample(int(x)) for x in layers])
    assert (many == one).all()


def test_session_streams_match_reference_logs():
    from benchlib.workloads import session_stream

    g = _sim()
    for s, lines in enumerate(g["sessions"]):
        recs = [json.loads(ln) for ln in lines]
        sid, stream = session_stream(g["questions"], g["queries_per_session"], g["seed"], s)
        assert sid == recs[0]["session_id"]
        assert [t for t, _ in stream] == [r["query_text"] for r in recs]
        assert [o for _, o in stream] == [r["origin"] for r in recs]
