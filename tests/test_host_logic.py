"""Host-side logic that needs no GPU: value types, config, embedder, sharding."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def test_hash_embedder_matches_reference_golden():
    from paper_2506_21593_b200 import HashEmbedder

    emb = HashEmbedder()
    with open(os.path.join(HERE, "golden", "embed.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        v = emb.embed(c["text"]).values
        nz = np.nonzero(v)[0]
        assert nz.tolist() == c["nz_index"], c["text"]
        assert v[nz].view(np.uint32).tolist() == c["nz_value_bits"], c["text"]


def test_answer_record_invariants_and_served_as():
    from paper_2506_21593_b200 import AnswerRecord, LayerTag

    a = AnswerRecord(text="x", layer=LayerTag.NAIVE_RAG, confidence=0.9, supporting_passage_ids=("p1",))
    kv = a.served_as(LayerTag.FIXED_KV, 0.0)
    assert kv.layer is LayerTag.FIXED_KV and kv.supporting_passage_ids == ()
    with pytest.raises(ValueError):
        AnswerRecord(text="x", layer=LayerTag.NAIVE_RAG, confidence=0.9)
    with pytest.raises(ValueError):
        AnswerRecord(text="x", layer=LayerTag.FIXED_KV, confidence=0.9, supporting_passage_ids=("p",))
    with pytest.raises(ValueError):
        AnswerRecord(text="x", layer=LayerTag.FIXED_KV, confidence=1.5)
    assert AnswerRecord.from_dict(a.to_dict()) == a
    assert LayerTag.from_wire("semantic_cache") is LayerTag.SEMANTIC_CACHE


def test_router_config_validation():
    from paper_2506_21593_b200 import LayerTag, RouterConfig

    with pytest.raises(ValueError):
        RouterConfig(semantic_threshold=0.0)
    with pytest.raises(ValueError):
        RouterConfig(recall_threshold=-0.1)
    with pytest.raises(ValueError):
        RouterConfig(retrieval_k=5, akm_seed_k=3)
    with pytest.raises(ValueError):
        RouterConfig(layer_order=(LayerTag.FIXED_KV,))
    cfg = RouterConfig(disabled_layers=frozenset({LayerTag.MEMORY_RECALL}))
    assert LayerTag.MEMORY_RECALL not in cfg.probe_order()


def test_validate_query_keeps_bytes():
    from paper_2506_21593_b200 import EmptyQuery, validate_query

    q = validate_query("  Who?  ", "s")
    assert q.text == "  Who?  "
    with pytest.raises(EmptyQuery):
        validate_query("   ", "s")


@pytest.mark.parametrize("n,world", [(10, 1), (10, 3), (7, 8), (10_000_000, 8), (0, 2)])
def test_shard_range_partitions(n, world):
    from paper_2506_21593_b200 import shard_range

    spans = [shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and b - a >= d - c >= b - a - 1


def test_vector_contract():
    from paper_2506_21593_b200 import DimensionMismatch, EmbeddingVector, InvalidVector
    from paper_2506_21593_b200.vectors import coerce_index_vector

    v = np.zeros(8, np.float32)
    v[0] = 1
    assert coerce_index_vector(v, 8).shape == (8,)
    with pytest.raises(InvalidVector):
        coerce_index_vector(np.ones(8, np.float32), 8)
    with pytest.raises(InvalidVector):
        coerce_index_vector(v[:4], 8)
    bad = v.copy()
    bad[1] = np.nan
    with pytest.raises(InvalidVector):
        coerce_index_vector(bad, 8)
    with pytest.raises(DimensionMismatch):
        EmbeddingVector.wrap(v)  # default dim 1024


def test_triples_reader_strict(tmp_path):
    """generation._read_triples follows ragcascade/jsonl.py:12-49: blank lines skipped,
    malformed JSON or a non-object raises MalformedJsonl with the 1-based line number."""
    from paper_2506_21593_b200 import MalformedJsonl
    from paper_2506_21593_b200.generation import _read_triples

    p = tmp_path / "ok.jsonl"
    p.write_text('{"question": "a", "answer": "b"}\n\n  \n{"question": "c", "answer": "d"}\n', encoding="utf-8")
    assert [o["question"] for o in _read_triples(p)] == ["a", "c"]
    for body, line in (('{"q": 1}\n{oops\n', 2), ('"str"\n', 1)):
        bad = tmp_path / "bad.jsonl"
        bad.write_text(body, encoding="utf-8")
        with pytest.raises(MalformedJsonl) as ei:
            _read_triples(bad)
        assert ei.value.line_number == line
