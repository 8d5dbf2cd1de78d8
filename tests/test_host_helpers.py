"""Host-side helpers of the batched cascade (CPU only)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2506_21593_b200.index import first_occurrences
from paper_2506_21593_b200.textarena import encode_texts


def test_first_occurrences_matches_unique():
    rng = np.random.default_rng(0)
    pos = np.empty(1000, dtype=np.int32)
    for _ in range(300):
        rows = rng.integers(0, int(rng.integers(1, 1000)), int(rng.integers(0, 400)))
        _, want = np.unique(rows, return_index=True)
        want.sort()
        assert first_occurrences(rows, pos).tolist() == want.tolist()


@pytest.mark.parametrize("texts", [[], ["a"], ["abc", "", "de"], ["é", "x", "日本"], ["\udc80", "ok"],
                                   [f"query-{i:09d}" for i in range(50)]])
def test_encode_texts_arena(texts):
    data, off = encode_texts(texts)
    bs = [t.encode("utf-8", "surrogatepass") for t in texts]
    assert off.dtype == np.int64 and off.tolist() == [0] + np.cumsum([len(b) for b in bs]).tolist()
    assert bytes(data[: off[-1]]) == b"".join(bs)
    assert data.size >= 1  # never an empty device buffer


def test_ctx_rows_slices_lazily():
    from paper_2506_21593_b200.ledger import CtxRows

    rows = np.arange(30, dtype=np.int64).reshape(3, 10)
    slot = np.array([2, -1, 0, 1])
    count = np.array([10, 2, 5], dtype=np.int32)  # per slot
    served = np.array([True, False, True, True])
    c = CtxRows(rows, slot, count, 3, served)
    assert c.get(0).tolist() == [20, 21, 22]
    assert c.get(1) is None
    assert c.get(2).tolist() == [0, 1, 2]
    assert c.get(3).tolist() == [10, 11]  # fewer than k results
