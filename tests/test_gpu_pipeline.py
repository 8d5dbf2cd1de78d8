"""pipeline.search_stream: streamed batches from pinned host memory give exactly the
per-batch search_batch results (rows, reported scores, counts), in order, with the copies
overlapped with the scans (double-buffered device / host buffers, event-ordered)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import random_unit_vectors

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("sharded", [False, True])
def test_search_stream_equals_search_batch(gpu, rng, sharded):
    import torch

    from paper_2506_21593_b200 import FlatIndex, ShardedFlatIndex
    from paper_2506_21593_b200.pipeline import search_stream

    d, n, k = 256, 600_000, 5  # large enough for the int8 path (>= 512k rows)
    X = random_unit_vectors(rng, n, d)
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"r{i}" for i in range(n)], X)
    index = ShardedFlatIndex(idx, 0) if sharded else idx
    batches = []
    for b, size in enumerate([300, 300, 77, 512, 300, 1]):
        Q = random_unit_vectors(rng, size, d)
        Q[0] = X[(b * 7919) % n]  # a self-snap per batch
        batches.append(torch.from_numpy(Q).pin_memory())
    want = []
    for hb in batches:
        r = idx.search_batch(hb.cuda(), k)
        want.append((r.rows.cpu().numpy(), r.scores.cpu().numpy(), r.count.cpu().numpy()))
    got = [tuple(t.numpy().copy() for t in res) for res in search_stream(index, batches, k)]
    assert len(got) == len(want)
    for b, (g, w) in enumerate(zip(got, want)):
        np.testing.assert_array_equal(g[0], w[0], err_msg=f"batch {b} rows")
        assert (g[1].view(np.int64) == w[1].view(np.int64)).all(), f"batch {b} score bits"
        np.testing.assert_array_equal(g[2], w[2], err_msg=f"batch {b} counts")
    assert list(search_stream(index, [], k)) == []
    # a consumer that stops after the first batch: the generator's cleanup waits for the
    # copy stream, and a fresh stream afterwards still gives the right answers
    first = next(iter(search_stream(index, batches, k)))
    np.testing.assert_array_equal(first[0].numpy(), want[0][0])
    again = [t[0].numpy().copy() for t in search_stream(index, batches[:2], k)]
    np.testing.assert_array_equal(again[1], want[1][0])
