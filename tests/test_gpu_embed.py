"""Device HashEmbedder == reference HashEmbedder bit-for-bit (embedding.py:117-160)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_device_embed_matches_reference_golden(gpu):
    from paper_2506_21593_b200 import HashEmbedder

    with open(os.path.join(HERE, "golden", "embed.json")) as fh:
        cases = json.load(fh)
    emb = HashEmbedder()
    V = emb.embed_device([c["text"] for c in cases]).cpu().numpy()
    for c, v in zip(cases, V):
        nz = np.nonzero(v)[0]
        assert nz.tolist() == c["nz_index"], c["text"]
        assert v[nz].view(np.uint32).tolist() == c["nz_value_bits"], c["text"]


def test_device_embed_matches_host_on_workload_texts(gpu):
    from benchlib.workloads import corpus_of, qa_rows, session_stream
    from paper_2506_21593_b200 import HashEmbedder

    rows = qa_rows(3000, 42)
    texts = [c["text"] for c in corpus_of(rows)]
    _, st = session_stream([r["question"] for r in rows], 3000, 0, 0)
    texts += [t for t, _ in st]
    texts += ["", "!!!", "x y x y", "a " * 300, "ünïcödé ✓", "tab\tand\nnewline", "under_score 42", "ß"]
    for dim in (1024, 384):
        emb = HashEmbedder(dim=dim)
        want = []
        for t in texts:
            try:
                want.append(emb.embed_array(t))
            except Exception:  # noqa: BLE001 - empty text
                want.append(None)
        ok_texts = [t for t, w in zip(texts, want) if w is not None]
        got = emb.embed_device(ok_texts).cpu().numpy()
        np.testing.assert_array_equal(got, np.stack([w for w in want if w is not None]))
    with pytest.raises(Exception):
        HashEmbedder().embed_device(["ok", ""])
