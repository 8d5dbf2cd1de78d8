"""pr_index_search_floor (FlatIndex.search_batch(floor=...)): the threshold-lookup search
of the semantic cache / adaptive memory (src/caches.py:140, src/knowledge.py:203-205).

Contract: every result whose exact score is >= min(floor, 1 - 1e-6) is exact and in its
exact rank; so `count > 0 and reported[0] >= floor` is exactly the full search's decision,
and on a hit the row and score bits are the full search's.  Checked against the exact fp64
path (itself bit-identical to the reference, tests/test_gpu_index.py) on near-duplicates,
random queries, stored-row copies (self-snap to 1.0), duplicated stored rows (ties), row
limits, and per-query floors at the exact top-1 score and its nextafter."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(rng, n, d, b):
    X = rng.standard_normal((n, d))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    X = X.astype(np.float32)
    X[n // 3] = X[n // 5]  # a duplicated row: an exact tie
    Q = rng.standard_normal((b, d))
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    nb = b // 3
    rows = rng.integers(0, n, nb)
    cos = rng.uniform(0.80, 0.995, (nb, 1))
    noise = rng.standard_normal((nb, d))
    base = X[rows].astype(np.float64)
    noise -= (noise * base).sum(1, keepdims=True) * base
    noise /= np.linalg.norm(noise, axis=1, keepdims=True)
    Q[:nb] = cos * base + np.sqrt(1 - cos ** 2) * noise
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    Q = Q.astype(np.float32)
    Q[nb:nb + 8] = X[rng.integers(0, n, 8)]  # stored-row copies: self-snap to 1.0
    Q[nb + 8] = X[n // 5]  # ... of the duplicated row
    return X, Q


def _decide(count, rep, floor):
    return (count > 0) & (rep[:, 0] >= floor)


@pytest.mark.parametrize("n,d", [(3000, 384), (60000, 1024), (300000, 768)])
@pytest.mark.parametrize("k", [1, 3])
def test_floor_search_matches_full_search(gpu, n, d, k):
    import torch

    from paper_2506_21593_b200 import MODE_AUTO, MODE_EXACT, MODE_TENSOR_I8, FlatIndex

    rng = np.random.default_rng(n + d + k)
    X, Q = _case(rng, n, d, 600)
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"r{i}" for i in range(n)], X)
    q = torch.from_numpy(Q).cuda()
    full = idx.search_batch(q, k, mode=MODE_EXACT)
    f_rows, f_raw, f_rep, f_cnt = (t.cpu().numpy() for t in (full.rows, full.raw, full.scores, full.count))
    lim = torch.from_numpy(rng.integers(n // 2, n + 1, len(Q))).cuda()
    full_l = idx.search_batch(q, k, mode=MODE_EXACT, row_limit=lim)
    l_rows, l_raw, l_rep, l_cnt = (t.cpu().numpy() for t in (full_l.rows, full_l.raw, full_l.scores, full_l.count))
    floors = [0.0, 0.5, 0.85, 0.9, 0.999, 1.0]
    # per-query boundary probes: the exact top-1 reported score (hit) and the next double (miss)
    top = np.where(f_cnt > 0, f_rep[:, 0], 0.0)
    for mode in (MODE_AUTO, MODE_TENSOR_I8):
        for fl in floors + ["top", "next"]:
            if fl == "top":
                sel = np.arange(0, len(Q), 7)
                fls = top[sel]
            elif fl == "next":
                sel = np.arange(0, len(Q), 7)
                fls = np.nextafter(top[sel], np.inf)
            else:
                sel = np.arange(len(Q))
                fls = np.full(len(sel), fl)
            for f in np.unique(fls):
                qi = sel[fls == f]
                for lim_on in (False, True):
                    got = idx.search_batch(q[torch.from_numpy(qi).cuda()], k, mode=mode, floor=float(f),
                                           row_limit=lim[torch.from_numpy(qi).cuda()] if lim_on else None)
                    g_rows, g_raw, g_rep, g_cnt = (t.cpu().numpy() for t in (got.rows, got.raw, got.scores, got.count))
                    rows_, raw_, rep_, cnt_ = (l_rows, l_raw, l_rep, l_cnt) if lim_on else (f_rows, f_raw, f_rep, f_cnt)
                    want_hit = _decide(cnt_[qi], rep_[qi], f)
                    got_hit = _decide(g_cnt, g_rep, f)
                    assert (want_hit == got_hit).all(), (mode, f, lim_on)
                    # every full result at or above the floor is reported, exactly, in rank
                    fe = min(float(f), 1.0 - 1e-6)
                    for j in range(k):
                        m = (cnt_[qi] > j) & (raw_[qi, j] >= fe)
                        assert (g_rows[m, j] == rows_[qi][m, j]).all(), (mode, f, j)
                        assert (g_raw[m, j].view(np.int64) == raw_[qi][m, j].view(np.int64)).all()
                        assert (g_rep[m, j].view(np.int64) == rep_[qi][m, j].view(np.int64)).all()


def test_floor_search_rejects_nan(gpu):
    import torch

    from paper_2506_21593_b200 import FlatIndex

    idx = FlatIndex(dim=64)
    idx.extend_arrays(["a"], np.eye(1, 64, dtype=np.float32))
    with pytest.raises(ValueError):
        idx.search_batch(torch.from_numpy(np.eye(1, 64, dtype=np.float32)).cuda(), 1, floor=float("nan"))
