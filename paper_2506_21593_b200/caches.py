"""Layer 1 (fixed KV cache) and layer 2 (semantic cache) on the GPU.

Drop-ins for ``ragcascade/caches.py``: ``FixedKVCache`` (:45-101),
``SemanticCache`` (:104-228) and ``writeback`` (:231-253), same methods,
counters and error behaviour.

* FixedKVCache keys libpentarag's open-addressing table by the query's UTF-8
  bytes (byte-exact: tag matches are confirmed against the stored key bytes,
  caches.py:57-58); the table value is the write sequence number, i.e. the
  index of the CacheEntry in a host arena, so "last write wins"
  (caches.py:67-74) is a device atomicMax.  ``get_batch`` hashes and probes a
  whole batch in one kernel (the L1 probe of a routed batch).
* SemanticCache keeps its entries in a device FlatIndex keyed by query text
  (upsert) and answers ``lookup`` with the exact top-1 + inclusive threshold
  (caches.py:131-145); ``lookup_batch`` does it for a [B, dim] batch.
"""
from __future__ import annotations

import ctypes
import logging
import threading
import time
from collections import OrderedDict
from dataclasses import dataclass
from typing import Any, Sequence

import numpy as np

from . import _lib
from .errors import CascadeError
from .index import MODE_AUTO, FlatIndex
from .records import AnswerRecord, Query
from .vectors import DIMENSION

log = logging.getLogger(__name__)

DEFAULT_SEMANTIC_THRESHOLD = 0.85


@dataclass(frozen=True)
class CacheEntry:
    query_text: str
    answer: AnswerRecord
    created_at_ns: int


from .textarena import encode_texts, to_device  # noqa: E402,F401  (encode_texts re-exported for callers)


def fingerprint_host(text: str) -> tuple[int, int]:
    L = _lib.load()
    b = text.encode("utf-8", "surrogatepass")
    buf = ctypes.create_string_buffer(b, max(1, len(b)))
    out = (ctypes.c_uint64 * 2)()
    L.pr_fingerprint_host(ctypes.cast(buf, ctypes.c_void_p), len(b), out)
    return int(out[0]), int(out[1])


class FixedKVCache:
    """Exact-match cache: raw query text -> last answer written.

    The device table (libpentarag ``pr_kv_*``) maps the key's bytes to an int64 write
    sequence number; the number indexes the host arena of written entries.  Hits are
    byte-exact (the table confirms every tag match against the stored key bytes).
    The host arena is compacted when overwritten / evicted entries make up half of it,
    so memory follows the live keys, not the write traffic (caches.py:75-77)."""

    _COMPACT_MIN = 4096

    def __init__(self, max_entries: int | None = None, *, capacity: int = 1024):
        if max_entries is not None and max_entries < 1:
            raise ValueError("max_entries must be >= 1 or None")
        _lib.require_device()
        self._L = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self._L.pr_kv_create(max(capacity, max_entries or 0), ctypes.byref(h)), "pr_kv_create")
        self._h = h
        self._max_entries = max_entries
        self._arena: list = []
        self._compact_at = self._COMPACT_MIN
        self._compact_hold = 0  # > 0 while a routed batch holds probe results (arena indices)
        self._recency: OrderedDict[str, None] = OrderedDict()
        self._lock = threading.Lock()
        self.hits = 0
        self.misses = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._L.pr_kv_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    # -- single-key surface (caches.py:57-89) -----------------------------
    def get(self, query_text: str) -> AnswerRecord | None:
        import torch

        arena = to_device([query_text])
        vals = torch.empty(1, dtype=torch.int64, device="cuda")
        hit = torch.empty(1, dtype=torch.uint8, device="cuda")
        with self._lock:
            _lib.check(self._L.pr_kv_get_text(self._h, _lib.ptr(arena[0]), _lib.ptr(arena[1]), 1, _lib.ptr(vals),
                                              _lib.ptr(hit), _lib.stream_ptr()), "kv_get")
            v = int(vals.item())
            if not int(hit.item()):
                self.misses += 1
                return None
            self.hits += 1
            return self._arena[v].answer

    def put(self, query_text: str, answer: AnswerRecord) -> None:
        self.put_many([query_text], [answer])

    def __bool__(self) -> bool:
        # an EMPTY store is still a store: the reference router injects stores with
        # ``kv_cache or FixedKVCache()`` (router.py:213-220), which would silently replace
        # an empty drop-in by a CPU store if emptiness made it falsy
        return True

    def __len__(self) -> int:
        with self._lock:
            return self._size()

    def _size(self) -> int:
        return int(self._L.pr_kv_size(self._h, _lib.stream_ptr()))

    def clear(self) -> None:
        with self._lock:
            _lib.check(self._L.pr_kv_clear(self._h, _lib.stream_ptr()), "kv_clear")
            self._arena.clear()
            self._compact_at = self._COMPACT_MIN
            self._recency.clear()

    def stats(self) -> dict[str, int]:
        with self._lock:
            return {"hits": self.hits, "misses": self.misses, "size": self._size()}

    def _live_seqs(self) -> np.ndarray:
        """Sorted write sequence numbers of every live key (synchronises)."""
        import torch

        n = self._size()
        while True:
            vals = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
            got = int(self._L.pr_kv_export(self._h, _lib.ptr(vals), n, _lib.stream_ptr()))
            if got < 0:
                _lib.check(got, "kv_export")
            if got <= n:
                return np.sort(vals[:got].cpu().numpy())
            n = got

    def export_entries(self) -> list[dict[str, Any]]:
        with self._lock:
            out = []
            for s in self._live_seqs().tolist():  # write order == OrderedDict order of the reference
                e = self._arena[s]
                out.append({"query_text": e.query_text, "answer": e.answer.to_dict(), "created_at_ns": e.created_at_ns})
            return out

    def _maybe_compact(self) -> None:
        """Drop arena entries no live key points at (overwritten or evicted), keeping
        write order; the device values are remapped in one kernel."""
        import torch

        if len(self._arena) < self._compact_at or self._compact_hold:
            return
        live = self._live_seqs()
        if 2 * live.size <= len(self._arena):
            remap = np.full(len(self._arena), -1, dtype=np.int64)
            remap[live] = np.arange(live.size, dtype=np.int64)
            d_map = torch.from_numpy(remap).cuda()
            _lib.check(self._L.pr_kv_remap(self._h, _lib.ptr(d_map), remap.size, _lib.stream_ptr()), "kv_remap")
            arena = self._arena
            self._arena = [arena[i] for i in live.tolist()]
        self._compact_at = max(self._COMPACT_MIN, 2 * len(self._arena))

    # -- batch surface ------------------------------------------------------
    def put_many(self, texts: Sequence[str], answers: Sequence[AnswerRecord]) -> None:
        """Sequential-equivalent bulk put (later writes of a key win)."""
        now = time.monotonic_ns()
        self.put_entries(texts, [CacheEntry(t, a, now) for t, a in zip(texts, answers)])

    def put_entries(self, texts: Sequence[str], entries: Sequence, *, arena=None) -> None:
        """Bulk put of prepared entries (CacheEntry or ledger.LedgerEntry).
        ``arena``: the ``DeviceTexts`` of a batch whose first ``len(texts)`` texts
        these are (skips re-encoding)."""
        import torch

        n = len(texts)
        if not n:
            return
        if arena is None:
            arena = to_device(texts)
        with self._lock:
            base = len(self._arena)
            self._arena.extend(entries)
            seq = torch.arange(base, base + n, dtype=torch.int64, device="cuda")
            s = _lib.stream_ptr()
            _lib.check(self._L.pr_kv_put_text(self._h, _lib.ptr(arena[0]), _lib.ptr(arena[1]), n, arena.nbytes_of(n),
                                              _lib.ptr(seq), s), "kv_put")
            if self._max_entries is not None:
                for t in texts:
                    self._recency.pop(t, None)
                    self._recency[t] = None
                evict = []
                while len(self._recency) > self._max_entries:
                    evict.append(self._recency.popitem(last=False)[0])
                if evict:
                    ea = to_device(evict)
                    _lib.check(self._L.pr_kv_erase_text(self._h, _lib.ptr(ea[0]), _lib.ptr(ea[1]), len(evict), s),
                               "kv_erase")
            self._maybe_compact()

    def probe_device(self, d_data, d_off, n: int):
        """Device-side batch probe: (values int64 [n], hit uint8 [n]) tensors.
        Counters are NOT updated (the caller accounts probes)."""
        import torch

        vals = torch.empty(n, dtype=torch.int64, device="cuda")
        hit = torch.empty(n, dtype=torch.uint8, device="cuda")
        if n:
            _lib.check(self._L.pr_kv_get_text(self._h, _lib.ptr(d_data), _lib.ptr(d_off), n, _lib.ptr(vals),
                                              _lib.ptr(hit), _lib.stream_ptr()), "kv_get_text")
        return vals, hit

    def get_batch(self, texts: Sequence[str]) -> list[AnswerRecord | None]:
        """Batched ``get``: one fingerprint+probe kernel for the whole batch."""
        arena = to_device(texts)
        with self._lock:
            vals, hit = self.probe_device(arena[0], arena[1], len(texts))
            vals, hit = vals.cpu().numpy(), hit.cpu().numpy()
            nh = int(hit.sum())
            self.hits += nh
            self.misses += len(texts) - nh
            return [self._arena[int(v)].answer if h else None for v, h in zip(vals, hit)]

    def entry_at(self, seq: int) -> CacheEntry:
        return self._arena[seq]


class SemanticCache:
    """Cosine-threshold cache over query embeddings (device FlatIndex)."""

    def __init__(self, embedder, threshold: float = DEFAULT_SEMANTIC_THRESHOLD, max_entries: int | None = None,
                 *, dim: int | None = None):
        if not 0.0 < threshold <= 1.0:
            raise ValueError(f"threshold {threshold} outside (0, 1]")
        if max_entries is not None and max_entries < 1:
            raise ValueError("max_entries must be >= 1 or None")
        self._embedder = embedder
        self.threshold = threshold
        self._max_entries = max_entries
        self._dim = dim or getattr(embedder, "dim", DIMENSION)
        self._index = FlatIndex(dim=self._dim)
        self._recency: dict[str, int] = {}
        self._seq = 0
        self._lock = threading.Lock()
        self.hits = 0
        self.misses = 0

    def lookup(self, query_embedding) -> tuple[AnswerRecord, float] | None:
        """Top-1 hit iff its reported score >= threshold (caches.py:131-145)."""
        index = self._index
        hits = index.search(query_embedding, k=1)
        with self._lock:
            if hits and hits[0].score >= self.threshold:
                self.hits += 1
                return index.payload(hits[0].entry_id).answer, hits[0].score
            self.misses += 1
            return None

    def lookup_batch(self, queries, *, mode: int = MODE_AUTO, account: bool = True):
        """Batched lookup over a [B, dim] tensor.  Returns device tensors
        (hit bool [B], row int64 [B], score float64 [B]); row and score are those of
        the exact top-1 for a hit (a miss may carry row -1).  The search only has to
        be exact at or above the threshold (``search_batch(floor=...)``), so the scan
        starts from the threshold as its bound."""
        index = self._index
        res = index.search_batch(queries, 1, mode=mode, floor=float(self.threshold))
        hit = (res.count > 0) & (res.scores[:, 0] >= self.threshold)
        if account:
            nh = int(hit.sum().item())
            with self._lock:
                self.hits += nh
                self.misses += int(hit.numel()) - nh
        return hit, res.rows[:, 0], res.scores[:, 0]

    def answer_at(self, row: int) -> AnswerRecord:
        return self._index.payload_at(row).answer

    def put(self, query_text: str, answer: AnswerRecord, vector=None) -> None:
        if vector is None:
            vector = self._embedder.embed(query_text)
        entry = CacheEntry(query_text=query_text, answer=answer, created_at_ns=time.monotonic_ns())
        with self._lock:
            self._index.insert(query_text, vector, entry)
            self._seq += 1
            self._recency[query_text] = self._seq
            if self._max_entries is not None and len(self._index) > self._max_entries:
                self._evict_locked()

    def _evict_locked(self) -> None:
        # rebuild from the most recently written entries, keeping their row order
        # (caches.py:166-181); rows move device-to-device, nothing is re-embedded
        keep = set(sorted(self._recency, key=self._recency.get, reverse=True)[: self._max_entries])
        old = self._index
        ids = [t for t in old.entry_ids() if t in keep]
        rows = [old.row_of(t) for t in ids]
        fresh = FlatIndex(dim=self._dim)
        fresh.append_rows_from(old, np.asarray(rows, dtype=np.int64), ids, [old.payload(t) for t in ids])
        fresh.search_count = old.search_count
        self._index = fresh
        self._recency = {t: self._recency[t] for t in keep}

    def __bool__(self) -> bool:
        # an EMPTY store is still a store: the reference router injects stores with
        # ``kv_cache or FixedKVCache()`` (router.py:213-220), which would silently replace
        # an empty drop-in by a CPU store if emptiness made it falsy
        return True

    def __len__(self) -> int:
        return len(self._index)

    def clear(self) -> None:
        with self._lock:
            self._index.clear()
            self._recency.clear()

    @property
    def index(self) -> FlatIndex:
        return self._index

    def stats(self) -> dict[str, Any]:
        return {"hits": self.hits, "misses": self.misses, "size": len(self._index)}

    def snapshot(self) -> bytes:
        return self._index.snapshot(payload_encoder=lambda e: {
            "query_text": e.query_text, "answer": e.answer.to_dict(), "created_at_ns": e.created_at_ns})

    @classmethod
    def restore(cls, data: bytes, embedder, threshold: float = DEFAULT_SEMANTIC_THRESHOLD,
                max_entries: int | None = None) -> "SemanticCache":
        restored = FlatIndex.restore(data, payload_decoder=lambda p: CacheEntry(
            query_text=p["query_text"], answer=AnswerRecord.from_dict(p["answer"]),
            created_at_ns=int(p["created_at_ns"])))
        cache = cls(embedder, threshold=threshold, max_entries=max_entries, dim=restored.dim)
        cache._index = restored
        for seq, text in enumerate(restored.entry_ids(), start=1):
            cache._recency[text] = seq
        cache._seq = len(cache._recency)
        return cache


def writeback(kv, sc, query: Query, answer: AnswerRecord, *, vector=None) -> None:
    """Write-through to both caches; failures are logged, never raised (caches.py:231-253)."""
    try:
        kv.put(query.text, answer)
    except CascadeError:
        log.exception("fixed KV write-back failed for query %s", query.id)
    try:
        sc.put(query.text, answer, vector=vector)
    except CascadeError:
        log.exception("semantic cache write-back failed for query %s", query.id)
