"""The int8 tcgen05 scan (PR_SEARCH_TENSOR_I8) vs the CPU oracle.

The int8 path scores with quantised rows/queries and a rigorous per-row error
bound, appends every row whose upper bound reaches the running k-th lower
bound, and rescores that complete candidate set in fp64 numpy-einsum order
(csrc/tc_scan_i8.cu).  Its results must equal the reference's bit for bit:
row ids, raw einsum scores and reported (snapped/clamped) scores
(reference index.py:155-189).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import random_unit_vectors
from test_gpu_index import _check, _store

pytestmark = pytest.mark.gpu


def _mode():
    from paper_2506_21593_b200 import MODE_TENSOR_I8

    return MODE_TENSOR_I8


@pytest.mark.parametrize("d", [64, 100, 384, 768, 1024])
@pytest.mark.parametrize("k", [1, 5, 10, 16])
def test_i8_matches_oracle(gpu, rng, d, k):
    from paper_2506_21593_b200 import FlatIndex

    n = 20000 + 77
    X = _store(rng, n, d)
    Q = random_unit_vectors(rng, 300, d)
    Q[0] = X[1]  # self-snap + duplicated rows (ties)
    Q[5] = X[n - 3]
    for i in range(10, 60):  # planted near-duplicates
        v = X[(i * 131) % n] + 0.05 * random_unit_vectors(rng, 1, d)[0]
        Q[i] = (v / np.linalg.norm(v.astype(np.float64))).astype(np.float32)
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, k, _mode())
    st = idx.stats()
    assert st.path == _mode()
    assert st.fallback == 0
    assert st.appended >= Q.shape[0] * k


def test_i8_one_hot_tie_tiers(gpu, rng):
    """One-hot rows: every query ties thousands of rows at the k-th score.
    Rows quantise exactly, so the window holds the whole tie tier; a tier
    larger than the per-query buffer goes to the exact rescan."""
    from paper_2506_21593_b200 import FlatIndex

    d, n = 64, 20000
    X = np.zeros((n, d), dtype=np.float32)
    X[np.arange(n), np.arange(n) % d] = 1.0
    Q = random_unit_vectors(rng, 130, d)
    Q[3] = X[5]
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, 10, _mode())


def test_i8_sparse_integer_rows_with_tiers(gpu, rng):
    """HashEmbedder-like rows (a handful of small integer counts, normalised):
    many bit-identical scores at the k-boundary, broken by lowest row."""
    from paper_2506_21593_b200 import FlatIndex

    d, n = 256, 30000
    C = np.zeros((n, d))
    for i in range(n):
        nz = rng.integers(2, 12)
        C[i, rng.integers(0, 24, nz)] += rng.choice([-1.0, 1.0], nz)
        if not C[i].any():
            C[i, 0] = 1.0
    X = (C / np.linalg.norm(C, axis=1, keepdims=True)).astype(np.float32)
    Qc = np.zeros((96, d))
    for i in range(96):
        Qc[i, rng.integers(0, 24, 6)] += 1.0
    Q = (Qc / np.linalg.norm(Qc, axis=1, keepdims=True)).astype(np.float32)
    Q[0] = X[17]
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    for k in (1, 3, 10):
        _check(idx, X, Q, k, _mode())


def test_i8_tie_tier_beyond_buffer(gpu, rng):
    from paper_2506_21593_b200 import FlatIndex

    d, n = 32, 60000
    X = random_unit_vectors(rng, n, d)
    X[5000:45000] = X[3]  # 40000 identical rows: more than the 32768-row buffer
    Q = random_unit_vectors(rng, 40, d)
    Q[0] = X[3]
    Q[1] = (X[3] + 0.01 * Q[1]) / np.linalg.norm((X[3] + 0.01 * Q[1]).astype(np.float64))
    Q = Q.astype(np.float32)
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, 10, _mode())
    assert idx.stats().fallback > 0


def test_i8_row_limits(gpu, rng):
    import torch

    from oracle import flat_index as F
    from paper_2506_21593_b200 import FlatIndex

    n, d = 9000, 64
    X = _store(rng, n, d)
    X[4000:4100] = X[50]
    Q = random_unit_vectors(rng, 130, d)
    Q[:10] = X[50]
    lim = rng.integers(0, n + 500, Q.shape[0])
    lim[0], lim[1], lim[2], lim[3] = 0, 51, 4050, 3
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    for k in (1, 5):
        res = idx.search_batch(torch.from_numpy(Q), k, mode=_mode(), row_limit=torch.from_numpy(lim))
        rows, raw, cnt = res.rows.cpu().numpy(), res.raw.cpu().numpy(), res.count.cpu().numpy()
        for b in range(Q.shape[0]):
            m = int(min(lim[b], n))
            want = F.search(X[:m], Q[b:b + 1], k)
            assert cnt[b] == want.count[0], b
            c = int(want.count[0])
            np.testing.assert_array_equal(rows[b, :c], want.rows[0, :c], err_msg=f"q{b} lim {lim[b]}")
            np.testing.assert_array_equal(raw[b, :c], want.raw[0, :c])


def test_i8_store_maintenance(gpu, rng):
    """truncate / clear / in-place upsert / append_from keep the int8 copy and
    its per-row bounds in step with the fp32 rows."""
    import torch

    from oracle import flat_index as F
    from paper_2506_21593_b200 import FlatIndex

    d = 128
    X = random_unit_vectors(rng, 30000, d)
    Q = random_unit_vectors(rng, 64, d)
    Q[0] = X[25000]
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(30000)], X)
    idx.truncate(20000)
    res = idx.search_batch(torch.from_numpy(Q), 5, mode=_mode())
    np.testing.assert_array_equal(res.rows.cpu().numpy(), F.search(X[:20000], Q, 5).rows)
    idx.clear()
    Y = random_unit_vectors(rng, 5000, d)
    idx.extend_arrays([f"f{i}" for i in range(5000)], Y)
    idx.insert("f7", Q[3])
    Y[7] = Q[3]
    res = idx.search_batch(torch.from_numpy(Q), 3, mode=_mode())
    np.testing.assert_array_equal(res.rows.cpu().numpy(), F.search(Y, Q, 3).rows)
    assert res.rows[3, 0].item() == 7 and res.scores[3, 0].item() == 1.0
    # device-to-device gather (AKM settle from KB rows)
    other = FlatIndex(dim=d)
    src_rows = np.array([4, 9, 7, 4000, 12], dtype=np.int64)
    other.append_rows_from(idx, src_rows, [f"g{i}" for i in range(len(src_rows))], [None] * len(src_rows))
    res = other.search_batch(torch.from_numpy(Q), 2, mode=_mode())
    np.testing.assert_array_equal(res.rows.cpu().numpy(), F.search(Y[src_rows], Q, 2).rows)


def test_i8_unnormalised_rows(gpu, rng):
    """The bound uses the measured norms, so rows off the unit sphere
    (validate=False) are still ranked exactly."""
    import torch

    from oracle import flat_index as F
    from paper_2506_21593_b200 import FlatIndex

    d, n = 96, 12000
    X = random_unit_vectors(rng, n, d) * rng.uniform(0.25, 3.0, (n, 1)).astype(np.float32)
    X[100, :] = 0.0  # an all-zero row
    Q = random_unit_vectors(rng, 50, d)
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X, validate=False)
    res = idx.search_batch(torch.from_numpy(Q), 5, mode=_mode(), validate=False)
    want = F.search(X, Q, 5)
    np.testing.assert_array_equal(res.rows.cpu().numpy(), want.rows)
    np.testing.assert_array_equal(res.raw.cpu().numpy(), want.raw)


@pytest.mark.parametrize("k", [1, 5, 16])
@pytest.mark.parametrize("stride", ["8", "2"])
def test_i8_pilot_path(gpu, rng, k, stride, monkeypatch):
    """The pilot (every stride-th tile; the default 128 needs >= 1024 tiles, so the
    stride is forced here) must not change any result (incl. ties and row limits).
    Stride 2 makes the pilot's seeds the true top-k for most queries: the post
    kernel's first phase then selects only seed rows."""
    import torch

    monkeypatch.setenv("PR_I8_PILOT_STRIDE", stride)

    from oracle import flat_index as F
    from paper_2506_21593_b200 import FlatIndex

    d, n = 128, 100_003
    X = _store(rng, n, d)
    X[70000:70040] = X[5]  # a tie tier outside the pilot tiles, and row 5 inside tile 0 (a pilot tile)
    Q = random_unit_vectors(rng, 260, d)
    Q[0] = X[5]
    for i in range(10, 40):
        v = X[(i * 7919) % n] + 0.05 * random_unit_vectors(rng, 1, d)[0]
        Q[i] = (v / np.linalg.norm(v.astype(np.float64))).astype(np.float32)
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, k, _mode())
    assert idx.stats().fallback == 0
    lim = rng.integers(0, n + 10, Q.shape[0])
    lim[0], lim[1] = 70010, 3
    res = idx.search_batch(torch.from_numpy(Q), k, mode=_mode(), row_limit=torch.from_numpy(lim))
    rows, raw, cnt = res.rows.cpu().numpy(), res.raw.cpu().numpy(), res.count.cpu().numpy()
    for b in range(0, Q.shape[0], 7):
        m = int(min(lim[b], n))
        want = F.c_search(X[:m], Q[b:b + 1], k)
        assert cnt[b] == want.count[0], b
        c = int(want.count[0])
        np.testing.assert_array_equal(rows[b, :c], want.rows[0, :c], err_msg=f"q{b} lim {lim[b]}")
        np.testing.assert_array_equal(raw[b, :c], want.raw[0, :c])


def test_i8_pilot_one_hot(gpu, rng):
    from paper_2506_21593_b200 import FlatIndex

    d, n = 64, 70000
    X = np.zeros((n, d), dtype=np.float32)
    X[np.arange(n), np.arange(n) % d] = 1.0
    Q = random_unit_vectors(rng, 130, d)
    Q[3] = X[5]
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, 10, _mode())


@pytest.mark.parametrize("d", [1536, 2048])
def test_i8_wide_rows(gpu, rng, d):
    from paper_2506_21593_b200 import FlatIndex

    n = 9000
    X = _store(rng, n, d)
    Q = random_unit_vectors(rng, 70, d)
    Q[0] = X[1]
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, 7, _mode())
    assert idx.stats().path == _mode()


@pytest.mark.parametrize("n,nq", [(1, 1), (5, 3), (255, 1), (257, 129), (3000, 257)])
def test_i8_tiny_stores_and_odd_batches(gpu, rng, n, nq):
    """Stores smaller than one 256-row tile, one query, and query counts that are not
    a multiple of the 256-query SM-pair tile."""
    from paper_2506_21593_b200 import FlatIndex

    d = 64
    X = random_unit_vectors(rng, n, d)
    Q = random_unit_vectors(rng, nq, d)
    Q[0] = X[n // 2]
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    for k in (1, 5, 16):
        _check(idx, X, Q, k, _mode())


@pytest.mark.parametrize("env", [{}, {"PR_I8_ARES": "0"}, {"PR_I8_CG": "1"}, {"PR_I8_REFINE": "0"},
                                 {"PR_I8_PILOT_STRIDE": "4"}, {"PR_I8_PILOT_STRIDE": "2"}, {"PR_I8_MC": "2"},
                                 {"PR_I8_MC": "4"}, {"PR_I8_GUNION": "0"}, {"PR_I8_FAST": "1"},
                                 {"PR_I8_POST": "warp"}])
def test_i8_kernel_variants(gpu, rng, env, monkeypatch):
    """The scan variants behind the per-call knobs (streamed vs resident query tile,
    single-CTA vs 2-CTA MMA, refiner off, denser pilots, 1 (default) / 2 / 4 CTA pairs per
    multicast cluster, no refiner union bound, the single-level fast path, the
    warp-per-query post kernel) all give the oracle's answer."""
    from paper_2506_21593_b200 import FlatIndex

    for key, val in env.items():
        monkeypatch.setenv(key, val)
    d, n = 256, 70001
    X = _store(rng, n, d)
    X[40000:40050] = X[3]
    Q = random_unit_vectors(rng, 300, d)
    Q[0] = X[3]
    for i in range(10, 40):
        v = X[(i * 7919) % n] + 0.05 * random_unit_vectors(rng, 1, d)[0]
        Q[i] = (v / np.linalg.norm(v.astype(np.float64))).astype(np.float32)
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    for k in (1, 10):
        _check(idx, X, Q, k, _mode())


@pytest.mark.parametrize("mc", ["1", "2", "4"])
@pytest.mark.parametrize("nq", [1, 255, 257, 700, 1500])
def test_i8_multicast_cluster_padding(gpu, rng, mc, nq, monkeypatch):
    """Query-group counts that do not fill the last multicast cluster: its spare pairs load
    and multiply zero query tiles in lockstep and report nothing."""
    from paper_2506_21593_b200 import FlatIndex

    monkeypatch.setenv("PR_I8_MC", mc)
    d, n = 384, 90001
    X = _store(rng, n, d)
    Q = random_unit_vectors(rng, nq, d)
    Q[0] = X[77]
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"e{i}" for i in range(n)], X)
    _check(idx, X, Q, 5, _mode())
