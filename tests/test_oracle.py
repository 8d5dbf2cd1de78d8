"""The CPU oracle pinned against the reference's own outputs (CPU only).

tests/golden/*.npz|json were produced by running the real reference
(tests/golden/make_golden.py); here the oracle must reproduce them
bit-for-bit, and the C einsum-order emulation must equal numpy's einsum on
this host (the reduction order is a property of the numpy build).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

from conftest import random_unit_vectors

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _cases():
    with open(os.path.join(GOLD, "flat_index.json")) as fh:
        return json.load(fh)["flat_index_cases"]


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "flat_index.npz"))


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['name']}-d{c['d']}-n{c['n']}-k{c['k']}")
@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_oracle_matches_reference_golden(gold, case, impl):
    from oracle import flat_index as F

    nm = case["name"]
    X, Q, k = gold[f"{nm}_X"], gold[f"{nm}_Q"], case["k"]
    res = F.search(X, Q, k) if impl == "numpy" else F.c_search(X, Q, k, nthreads=2)
    np.testing.assert_array_equal(res.count, gold[f"{nm}_count"])
    for b in range(Q.shape[0]):
        c = int(gold[f"{nm}_count"][b])
        np.testing.assert_array_equal(res.rows[b, :c], gold[f"{nm}_rows"][b, :c])
        np.testing.assert_array_equal(res.reported[b, :c], gold[f"{nm}_scores"][b, :c])


@pytest.mark.parametrize("d", [1, 2, 3, 4, 7, 8, 9, 13, 16, 64, 100, 384, 768, 1000, 1001, 1023, 1024])
def test_c_einsum_order_equals_numpy_einsum(d):
    """The reduction order the GPU rescoring reproduces == this host's numpy."""
    from oracle import flat_index as F

    rng = np.random.default_rng(d)
    X = random_unit_vectors(rng, 257, d)
    q = random_unit_vectors(rng, 1, d)[0]
    want = np.einsum("ij,j->i", X.astype(np.float64), q.astype(np.float64))
    np.testing.assert_array_equal(F.c_scores(X, q), want)


def test_einsum_chunk_invariance():
    from oracle import flat_index as F

    rng = np.random.default_rng(5)
    X = random_unit_vectors(rng, 5000, 96)
    q = random_unit_vectors(rng, 1, 96)[0]
    full = np.einsum("ij,j->i", X.astype(np.float64), q.astype(np.float64))
    chunked = F.einsum_scores_chunked([X[:1234], X[1234:4000], X[4000:]], q)
    np.testing.assert_array_equal(full, chunked)


def test_numpy_and_c_oracles_agree_with_ties_and_snap():
    from oracle import flat_index as F

    rng = np.random.default_rng(9)
    X = random_unit_vectors(rng, 2000, 48)
    X[10] = X[3]
    X[1999] = X[3]
    Q = random_unit_vectors(rng, 6, 48)
    Q[2] = X[3]
    for k in (1, 3, 10, 64):
        a, b = F.search(X, Q, k), F.c_search(X, Q, k)
        np.testing.assert_array_equal(a.rows, b.rows)
        np.testing.assert_array_equal(a.raw, b.raw)
        np.testing.assert_array_equal(a.reported, b.reported)
    assert list(F.search(X, Q, 3).rows[2]) == [3, 10, 1999]
    assert F.search(X, Q, 3).reported[2][0] == 1.0


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted")
def test_oracle_vs_live_reference_random():
    """Where the reference is importable (the build container), check the
    oracle against it on fresh seeded stores too."""
    sys.path.insert(0, "/root/reference/pkg/src")
    import ragcascade as rc

    from oracle import flat_index as F

    rng = np.random.default_rng(77)
    for d, n in [(8, 300), (1024, 400), (33, 50)]:
        X = random_unit_vectors(rng, n, d)
        X[5] = X[1]
        idx = rc.FlatIndex(dim=d)
        for i in range(n):
            idx.insert(f"e{i}", X[i])
        Q = random_unit_vectors(rng, 4, d)
        Q[0] = X[1]
        res = F.search(X, Q, 10)
        for b in range(4):
            hits = idx.search(Q[b], k=10)
            assert [int(h.entry_id[1:]) for h in hits] == list(res.rows[b, : len(hits)])
            assert [h.score for h in hits] == list(res.reported[b, : len(hits)])
