"""Vector contract of the hot path (reference: embedding.py:30-160).

``EmbeddingVector`` is a read-only float32 unit vector; ``cosine`` is the
fp64 dot clamped to [-1, 1]; ``HashEmbedder`` is the deterministic keyed
blake2b feature-hash embedder the reference uses for its workloads (kept on
the host here — the device embedder is the next row).

``DIMENSION`` defaults to the reference's 1024 but every store takes an
explicit ``dim`` (the C1/C2 configs use 384/768), so no monkey-patching of a
module constant is needed.
"""
from __future__ import annotations

import re
from dataclasses import dataclass
from hashlib import blake2b
from typing import Iterable, Protocol, Sequence

import numpy as np

from .errors import DimensionMismatch, EmptyInput, InvalidVector

DIMENSION = 1024
HASH_SEED = 0x5EED_1024_CA5C_ADE5
NORM_TOLERANCE = 1e-5          # embedder contract (embedding.py:36)
INDEX_NORM_TOLERANCE = 1e-4    # index boundary (index.py:46)

_WORD = re.compile(r"\w+", re.UNICODE)


def tokenize(text: str) -> list[str]:
    return _WORD.findall(text)


def _unit_check(arr: np.ndarray, dim: int, tol: float, shape_error=DimensionMismatch) -> None:
    if arr.shape != (dim,):
        raise shape_error(f"expected shape ({dim},), got {arr.shape}")
    if not np.isfinite(arr).all():
        raise InvalidVector("vector contains NaN or Inf components")
    norm = float(np.linalg.norm(arr.astype(np.float64)))
    if abs(norm - 1.0) > tol:
        raise InvalidVector(f"vector norm {norm} deviates from 1 by > {tol}")


@dataclass(frozen=True, eq=False)
class EmbeddingVector:
    values: np.ndarray

    @classmethod
    def wrap(cls, values, dim: int = DIMENSION) -> "EmbeddingVector":
        arr = np.array(values, dtype=np.float32, copy=True)
        _unit_check(arr, dim, NORM_TOLERANCE)
        arr.setflags(write=False)
        return cls(values=arr)

    @classmethod
    def normalized(cls, values, dim: int = DIMENSION) -> "EmbeddingVector":
        arr = np.asarray(values, dtype=np.float64)
        if arr.shape != (dim,):
            raise DimensionMismatch(f"expected {dim} components, got shape {arr.shape}")
        if not np.isfinite(arr).all():
            raise InvalidVector("vector contains NaN or Inf components")
        n = float(np.linalg.norm(arr))
        if n == 0.0:
            raise InvalidVector("cannot normalize a zero vector")
        return cls.wrap((arr / n).astype(np.float32), dim)

    def __len__(self) -> int:
        return int(self.values.shape[0])


def as_f32(vector) -> np.ndarray:
    """Accept an EmbeddingVector from either package (duck-typed) or an array."""
    vals = getattr(vector, "values", vector)
    return np.asarray(vals, dtype=np.float32)


def coerce_index_vector(vector, dim: int) -> np.ndarray:
    """The index-boundary check (index.py:58-70): shape, finite, |‖v‖-1| <= 1e-4."""
    arr = as_f32(vector)
    _unit_check(arr, dim, INDEX_NORM_TOLERANCE, shape_error=InvalidVector)
    return arr


def cosine(a, b) -> float:
    va, vb = as_f32(a), as_f32(b)
    if va.shape != vb.shape:
        raise DimensionMismatch(f"shapes differ: {va.shape} vs {vb.shape}")
    s = float(np.dot(va.astype(np.float64), vb.astype(np.float64)))
    return min(1.0, max(-1.0, s))


class Embedder(Protocol):
    def embed(self, text: str) -> EmbeddingVector: ...

    def embed_many(self, texts: Sequence[str]) -> list[EmbeddingVector]: ...


class HashEmbedder:
    """Bag-of-tokens feature hashing: bucket = h % dim, sign = bit 63 of a keyed
    64-bit blake2b of ``b"tok:" + token``; fp64 accumulate, L2 normalise, fp32.
    Texts whose signs cancel fall back to a one-hot from ``b"raw:" + text``."""

    def __init__(self, seed: int = HASH_SEED, dim: int = DIMENSION):
        self.dim = dim
        self._key = seed.to_bytes(8, "big")
        self._memo: dict[str, tuple[int, float]] = {}

    def _h(self, data: bytes) -> int:
        return int.from_bytes(blake2b(data, digest_size=8, key=self._key).digest(), "big")

    def _slot(self, tok: str) -> tuple[int, float]:
        hit = self._memo.get(tok)
        if hit is None:
            h = self._h(b"tok:" + tok.encode("utf-8"))
            hit = (h % self.dim, 1.0 if h >> 63 else -1.0)
            self._memo[tok] = hit
        return hit

    def embed_array(self, text: str) -> np.ndarray:
        if not text:
            raise EmptyInput("cannot embed an empty string")
        acc = np.zeros(self.dim, dtype=np.float64)
        for tok in tokenize(text):
            b, s = self._slot(tok)
            acc[b] += s
        n = float(np.linalg.norm(acc))
        if n == 0.0:
            h = self._h(b"raw:" + text.encode("utf-8"))
            out = np.zeros(self.dim, dtype=np.float32)
            out[h % self.dim] = 1.0 if h >> 63 else -1.0
            return out
        return (acc / n).astype(np.float32)

    def embed(self, text: str) -> EmbeddingVector:
        return EmbeddingVector.wrap(self.embed_array(text), self.dim)

    def embed_many(self, texts: Sequence[str]) -> list[EmbeddingVector]:
        return [self.embed(t) for t in texts]

    def embed_matrix(self, texts: Iterable[str]) -> np.ndarray:
        return np.stack([self.embed_array(t) for t in texts]) if texts else np.zeros((0, self.dim), np.float32)

    def embed_device(self, texts, *, arena=None) -> "object":
        """Embed a batch on the GPU (libpentarag pr_hash_embed: keyed BLAKE2b token
        hashing, warp per text) into a float32 CUDA tensor [n, dim], bit-identical
        to ``embed``.  The device takes every non-empty ASCII text of at most 512
        characters (so at most 256 tokens); the others are picked out on the host
        BEFORE the launch, embedded there and patched in — no device-to-host read, so
        the call never waits for the GPU.  An empty text raises EmptyInput exactly
        like ``embed``."""
        import torch

        from . import _lib
        from .textarena import to_device

        texts = list(texts)
        n = len(texts)
        out = torch.empty((n, self.dim), dtype=torch.float32, device="cuda")
        if n == 0:
            return out
        d_data, d_off = arena if arena is not None else to_device(texts)  # arena: the texts' device UTF-8 arena
        flag = torch.empty(n, dtype=torch.uint8, device="cuda")
        L = _lib.load()
        _lib.check(L.pr_hash_embed(_lib.ptr(d_data), _lib.ptr(d_off), n, self.dim, int.from_bytes(self._key, "big"),
                                   _lib.ptr(out), _lib.ptr(flag), _lib.stream_ptr()), "hash_embed")
        if getattr(arena, "ascii", None):  # all ASCII: a text's byte count is its length
            lens = np.diff(arena.host_off)
            host = np.flatnonzero((lens == 0) | (lens > 512)).tolist()
        else:
            host = [i for i, t in enumerate(texts) if not (t and t.isascii() and len(t) <= 512)]
        if host:
            rows = np.stack([self.embed_array(texts[i]) for i in host])
            out[torch.tensor(host, device="cuda")] = torch.from_numpy(rows).cuda()
        return out


def mean_cosine(reference, others: Iterable) -> float:
    vals = [cosine(reference, o) for o in others]
    if not vals:
        raise ValueError("mean_cosine needs at least one comparison vector")
    return float(np.mean(vals))
