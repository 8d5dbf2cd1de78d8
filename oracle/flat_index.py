"""TEST INFRASTRUCTURE ONLY — restatement of ``FlatIndex.search``.

Reference: /root/reference/pkg/src/ragcascade/index.py:155-189.  The scan is
``np.einsum("ij,j->i", V64, q64)`` (index.py:173) over float32 rows upcast to
float64 (index.py:145), ranking by ``np.lexsort((arange(n), -scores))``
(index.py:176), then per hit the self-snap (index.py:180-181) and the clamp
(index.py:185).  This module calls the very same numpy routines, so on the
same numpy build it is bit-identical to the reference by construction; the C
twin (einsum_order.c) re-derives the reduction order independently.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")


@dataclass
class OracleResult:
    rows: np.ndarray       # int64 [B, k], -1 where count < k
    raw: np.ndarray        # float64 [B, k] — einsum score before snap/clamp
    reported: np.ndarray   # float64 [B, k] — SearchHit.score
    count: np.ndarray      # int32 [B]


def _finish(X32: np.ndarray, q32: np.ndarray, order: np.ndarray, scores: np.ndarray, k: int):
    rows = np.full(k, -1, dtype=np.int64)
    raw = np.zeros(k)
    rep = np.zeros(k)
    for rank, row in enumerate(order):
        s = float(scores[row])
        rows[rank] = row
        raw[rank] = s
        if s > 1.0 - 1e-6 and np.array_equal(X32[row], q32):      # index.py:180-181
            s = 1.0
        rep[rank] = max(-1.0, min(1.0, s))                          # index.py:185
    return rows, raw, rep


def search(X32: np.ndarray, Q32: np.ndarray, k: int) -> OracleResult:
    """numpy restatement of FlatIndex.search for each row of ``Q32``."""
    if k < 1:
        raise ValueError("k must be >= 1")
    X32 = np.ascontiguousarray(X32, dtype=np.float32)
    Q32 = np.atleast_2d(np.ascontiguousarray(Q32, dtype=np.float32))
    n = X32.shape[0]
    B = Q32.shape[0]
    out = OracleResult(
        rows=np.full((B, k), -1, dtype=np.int64),
        raw=np.zeros((B, k)),
        reported=np.zeros((B, k)),
        count=np.zeros(B, dtype=np.int32),
    )
    if n == 0:
        return out
    X64 = X32.astype(np.float64)                                      # index.py:145
    take = min(k, n)
    for b in range(B):
        q64 = Q32[b].astype(np.float64)
        scores = np.einsum("ij,j->i", X64, q64)                       # index.py:173
        order = np.lexsort((np.arange(n), -scores))[:take]            # index.py:176
        out.rows[b], out.raw[b], out.reported[b] = _finish(X32, Q32[b], order, scores, k)
        out.count[b] = take
    return out


def einsum_scores_chunked(chunks, q32: np.ndarray) -> np.ndarray:
    """Scores of one query over a store given as an iterable of float32 row
    chunks.  einsum is a per-row reduction, so chunking never changes a
    score bit (verified in tests/test_oracle.py)."""
    q64 = np.asarray(q32, dtype=np.float32).astype(np.float64)
    return np.concatenate(
        [np.einsum("ij,j->i", np.asarray(c, dtype=np.float32).astype(np.float64), q64) for c in chunks]
    )


def topk_from_scores(scores: np.ndarray, k: int) -> np.ndarray:
    n = scores.shape[0]
    return np.lexsort((np.arange(n), -scores))[: min(k, n)]


# --- C twin ---------------------------------------------------------------

_lib = None


def lib():
    """ctypes handle on oracle/_build/liboracle.so (built by `make -C oracle`)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            import subprocess

            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_einsum_dot.restype = ctypes.c_double
        L.oracle_einsum_dot.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_scores.restype = None
        L.oracle_scores.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_search.restype = ctypes.c_int
        L.oracle_search.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
        ]
        L.oracle_pair_scores.restype = None
        L.oracle_pair_scores.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int64, ctypes.c_void_p,
        ]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def c_scores(X32: np.ndarray, q32: np.ndarray) -> np.ndarray:
    X32 = np.ascontiguousarray(X32, dtype=np.float32)
    q32 = np.ascontiguousarray(q32, dtype=np.float32)
    out = np.empty(X32.shape[0])
    lib().oracle_scores(_p(X32), X32.shape[0], X32.shape[1], _p(q32), _p(out))
    return out


def c_search(X32: np.ndarray, Q32: np.ndarray, k: int, nthreads: int | None = None) -> OracleResult:
    """The C twin of :func:`search` (same semantics, pthreads over queries)."""
    X32 = np.ascontiguousarray(X32, dtype=np.float32)
    Q32 = np.ascontiguousarray(np.atleast_2d(Q32), dtype=np.float32)
    B, d = Q32.shape
    n = X32.shape[0] if X32.size else 0
    res = OracleResult(
        rows=np.empty((B, k), dtype=np.int64),
        raw=np.empty((B, k)),
        reported=np.empty((B, k)),
        count=np.empty(B, dtype=np.int32),
    )
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    rc = lib().oracle_search(
        _p(X32), n, d, _p(Q32), B, k, _p(res.rows), _p(res.raw), _p(res.reported), _p(res.count), nthreads
    )
    if rc != 0:
        raise ValueError("oracle_search rejected its arguments")
    return res


def c_pair_scores(X32, Q32, qidx, ridx) -> np.ndarray:
    X32 = np.ascontiguousarray(X32, dtype=np.float32)
    Q32 = np.ascontiguousarray(Q32, dtype=np.float32)
    qidx = np.ascontiguousarray(qidx, dtype=np.int64)
    ridx = np.ascontiguousarray(ridx, dtype=np.int64)
    out = np.empty(qidx.shape[0])
    lib().oracle_pair_scores(_p(X32), X32.shape[1], _p(Q32), _p(qidx), _p(ridx), qidx.shape[0], _p(out))
    return out
