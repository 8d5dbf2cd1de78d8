"""FlatIndex on the GPU vs the CPU oracle (reference index.py:155-189).

Bit-exact: row ids, raw fp64 scores (numpy einsum order) and reported
scores (snap + clamp) must equal the oracle's, in both the exact fp64 scan
and the tcgen05 fp16 scan + certified rescoring.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import random_unit_vectors

pytestmark = pytest.mark.gpu


def _oracle():
    from oracle import flat_index

    return flat_index


def _check(idx, X, Q, k, mode):
    import torch

    F = _oracle()
    res = idx.search_batch(torch.from_numpy(Q), k, mode=mode)
    torch.cuda.synchronize()
    want = F.c_search(X, Q, k)
    got_rows = res.rows.cpu().numpy()
    got_raw = res.raw.cpu().numpy()
    got_rep = res.scores.cpu().numpy()
    got_cnt = res.count.cpu().numpy()
    np.testing.assert_array_equal(got_cnt, want.count)
    for b in range(Q.shape[0]):
        c = want.count[b]
        np.testing.assert_array_equal(got_rows[b, :c], want.rows[b, :c], err_msg=f"query {b} rows")
        np.testing.assert_array_equal(got_raw[b, :c], want.raw[b, :c], err_msg=f"query {b} raw")
        np.testing.assert_array_equal(got_rep[b, :c], want.reported[b, :c], err_msg=f"query {b} reported")
    return res


def _store(rng, n, d, dup=True):
    X = random_unit_vectors(rng, n, d)
    if dup and n >= 4:
        X[n // 2] = X[1]
        X[n - 1] = X[1]
    return X


@pytest.mark.parametrize("d", [4, 8, 13, 64, 384, 768, 1024])
@pytest.mark.parametrize("k", [1, 3, 10])
def test_exact_matches_oracle(gpu, rng, d, k):
    from paper_2506_21593_b200 import MODE_EXACT, FlatIndex

    n = 3000
    X = _store(rng, n, d)
    Q = random_unit_vectors(rng, 33, d)
    Q[0] = X[1]  # tie-heavy probe with self-snap
    Q[1] = X[7]
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, k, MODE_EXACT)


@pytest.mark.parametrize("d", [64, 384, 768, 1024, 100])
@pytest.mark.parametrize("k", [1, 5, 10])
def test_tensor_path_matches_oracle(gpu, rng, d, k):
    from paper_2506_21593_b200 import MODE_TENSOR, FlatIndex

    n = 20000 + 77
    X = _store(rng, n, d)
    Q = random_unit_vectors(rng, 300, d)
    Q[0] = X[1]
    Q[5] = X[n - 3]
    # planted near-duplicates
    for i in range(10, 60):
        v = X[(i * 131) % n] + 0.05 * random_unit_vectors(rng, 1, d)[0]
        Q[i] = (v / np.linalg.norm(v.astype(np.float64))).astype(np.float32)
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, k, MODE_TENSOR)
    st = idx.stats()
    assert st.path == MODE_TENSOR
    assert st.fallback < Q.shape[0]


def test_tensor_path_fallback_on_ties(gpu, rng):
    """Massive exact ties (one-hot rows) defeat the certificate; the exact
    rescan must still give the oracle's answer."""
    from paper_2506_21593_b200 import MODE_TENSOR, FlatIndex

    d, n = 64, 20000
    X = np.zeros((n, d), dtype=np.float32)
    X[np.arange(n), np.arange(n) % d] = 1.0
    Q = random_unit_vectors(rng, 130, d)
    Q[3] = X[5]
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, 10, MODE_TENSOR)
    st = idx.stats()
    assert st.collected > 0  # ties defeat the certificate -> tcgen05 collect pass


def test_tensor_path_tie_tier_beyond_collect_cap(gpu, rng):
    """A tie tier larger than the collect capacity (8192 rows) must end in the
    exact fp64 rescan and still match the oracle (lowest rows win ties)."""
    from paper_2506_21593_b200 import MODE_TENSOR, FlatIndex

    d, n = 32, 30000
    X = random_unit_vectors(rng, n, d)
    X[5000:25000] = X[3]  # 20000 identical rows
    Q = random_unit_vectors(rng, 40, d)
    Q[0] = X[3]
    Q[1] = (X[3] + 0.01 * Q[1]) / np.linalg.norm((X[3] + 0.01 * Q[1]).astype(np.float64))
    Q = Q.astype(np.float32)
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, 10, MODE_TENSOR)
    assert idx.stats().fallback > 0


def test_empty_and_small(gpu, rng):
    from paper_2506_21593_b200 import MODE_AUTO, MODE_EXACT, FlatIndex

    idx = FlatIndex(dim=8)
    q = random_unit_vectors(rng, 1, 8)[0]
    assert idx.search(q, 5) == []
    assert idx.search_count == 1
    idx.insert("a", np.eye(8, dtype=np.float32)[0])
    idx.insert("b", np.eye(8, dtype=np.float32)[1])
    hits = idx.search(np.eye(8, dtype=np.float32)[0], 10)
    assert [(h.entry_id, h.score, h.rank) for h in hits] == [("a", 1.0, 1), ("b", 0.0, 2)]
    with pytest.raises(ValueError):
        idx.search(q, 0)


def test_upsert_keeps_row(gpu, rng):
    from paper_2506_21593_b200 import FlatIndex

    idx = FlatIndex(dim=16)
    vs = random_unit_vectors(rng, 3, 16)
    idx.insert("x", vs[0], 1)
    idx.insert("y", vs[1], 2)
    idx.insert("x", vs[1], 3)  # now x and y hold the same vector; x keeps row 0
    hits = idx.search(vs[1], 2)
    assert [h.entry_id for h in hits] == ["x", "y"]
    assert hits[0].score == 1.0
    assert idx.payload("x") == 3 and len(idx) == 2


@pytest.mark.parametrize("mode,k", [(1, 5), (2, 5), (2, 1), (0, 80)])
def test_row_limits_match_prefix_oracle(gpu, rng, mode, k):
    """pr_index_search_ex: query q must see exactly rows [0, limit[q])."""
    import torch

    from oracle import flat_index as F
    from paper_2506_21593_b200 import FlatIndex

    n, d = 9000, 64
    X = _store(rng, n, d)
    X[4000:4100] = X[50]  # ties straddling some limits
    Q = random_unit_vectors(rng, 130, d)
    Q[:10] = X[50]
    lim = rng.integers(0, n + 500, Q.shape[0])
    lim[0], lim[1], lim[2] = 0, 51, 4050
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    res = idx.search_batch(torch.from_numpy(Q), k, mode=mode, row_limit=torch.from_numpy(lim))
    rows, raw, cnt = res.rows.cpu().numpy(), res.raw.cpu().numpy(), res.count.cpu().numpy()
    for b in range(Q.shape[0]):
        m = int(min(lim[b], n))
        want = F.search(X[:m], Q[b:b + 1], k)
        assert cnt[b] == want.count[0], b
        c = int(want.count[0])
        np.testing.assert_array_equal(rows[b, :c], want.rows[0, :c], err_msg=f"q{b} lim {lim[b]}")
        np.testing.assert_array_equal(raw[b, :c], want.raw[0, :c])


def test_truncate_and_clear_hide_stale_rows(gpu, rng):
    import torch

    from oracle import flat_index as F
    from paper_2506_21593_b200 import MODE_EXACT, MODE_TENSOR, FlatIndex

    d = 128
    X = random_unit_vectors(rng, 30000, d)
    Q = random_unit_vectors(rng, 64, d)
    Q[0] = X[25000]  # only present in the truncated tail
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(30000)], X)
    idx.truncate(20000)
    for mode in (MODE_EXACT, MODE_TENSOR):
        res = idx.search_batch(torch.from_numpy(Q), 5, mode=mode)
        want = F.search(X[:20000], Q, 5)
        np.testing.assert_array_equal(res.rows.cpu().numpy(), want.rows)
    idx.clear()
    Y = random_unit_vectors(rng, 5000, d)
    idx.extend_arrays([f"f{i}" for i in range(5000)], Y)
    res = idx.search_batch(torch.from_numpy(Q), 5, mode=MODE_TENSOR)
    np.testing.assert_array_equal(res.rows.cpu().numpy(), F.search(Y, Q, 5).rows)
    # in-place update (upsert) is visible to both copies (fp32 exact + fp16 scan)
    idx.insert("f7", Q[3])
    Y[7] = Q[3]
    res = idx.search_batch(torch.from_numpy(Q), 3, mode=MODE_TENSOR)
    np.testing.assert_array_equal(res.rows.cpu().numpy(), F.search(Y, Q, 3).rows)
    assert res.rows[3, 0].item() == 7 and res.scores[3, 0].item() == 1.0


def test_tensor_request_with_large_k_and_empty_batch(gpu, rng):
    import torch

    from paper_2506_21593_b200 import MODE_TENSOR, FlatIndex

    X = _store(rng, 20000, 64)
    Q = random_unit_vectors(rng, 9, 64)
    idx = FlatIndex(dim=64)
    idx.extend_arrays([f"e{i}" for i in range(20000)], X)
    _check(idx, X, Q, 40, MODE_TENSOR)  # k > 16 candidates/split: exact path serves it
    res = idx.search_batch(torch.zeros((0, 64)), 5, mode=MODE_TENSOR)
    assert res.rows.shape == (0, 5)


def test_big_k(gpu, rng):
    from paper_2506_21593_b200 import FlatIndex

    X = _store(rng, 500, 32)
    Q = random_unit_vectors(rng, 4, 32)
    idx = FlatIndex(dim=32)
    idx.extend_arrays([f"e{i}" for i in range(500)], X)
    _check(idx, X, Q, 100, 0)
    _check(idx, X, Q, 700, 0)  # k > n truncates


def test_shared_index_across_streams(gpu, rng):
    """One index searched concurrently from two threads on two CUDA streams (e.g.
    routers sharing a knowledge base): each search waits for the previous one's
    scratch, so every answer equals the single-stream answer."""
    import threading

    import torch

    from paper_2506_21593_b200 import MODE_TENSOR, MODE_TENSOR_I8, FlatIndex

    d, n = 128, 40000
    X = _store(rng, n, d)
    Qa = torch.from_numpy(random_unit_vectors(rng, 300, d)).cuda()
    Qb = torch.from_numpy(random_unit_vectors(rng, 200, d)).cuda()
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    for mode in (MODE_TENSOR_I8, MODE_TENSOR):
        want_a = idx.search_batch(Qa, 5, mode=mode).rows.cpu()
        want_b = idx.search_batch(Qb, 7, mode=mode).rows.cpu()
        errors = []

        def worker(Q, k, want):
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(15):
                    got = idx.search_batch(Q, k, mode=mode).rows
                    s.synchronize()
                    if not bool((got.cpu() == want).all()):
                        errors.append(k)

        ts = [threading.Thread(target=worker, args=(Qa, 5, want_a)), threading.Thread(target=worker, args=(Qb, 7, want_b))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errors, f"mode {mode}: {len(errors)} wrong answers under concurrent streams"
