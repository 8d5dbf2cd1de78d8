"""Device-resident exact flat index — drop-in for ``FlatIndex``.

Reference: ``ragcascade/index.py:73-261``.  Same method set (insert, extend,
search, clear, payload, vector, entry_ids, __len__, __contains__, dim,
search_count, snapshot/restore) and the same results bit-for-bit: scores are
the reference's fp64 ``np.einsum`` values (index.py:173) reproduced on the
GPU in numpy's reduction order, ranked by (score desc, row asc)
(index.py:176), self-snapped and clamped (index.py:180-185).

Ids and payloads stay in Python (they are opaque objects); vectors live in
libpentarag's device store (fp32 exact copy + fp16 tensor-core copy).  The
batch entry point ``search_batch`` takes a [B, dim] float32 tensor (device or
host) and returns device tensors; it is what the cascade and the benches use.
"""
from __future__ import annotations

import bisect
import weakref
import ctypes
import json
import struct
import threading
import zlib
from dataclasses import dataclass
from typing import Any, Callable, Iterable

import numpy as np

from . import _lib
from .errors import CorruptSnapshot, InvalidVector
from .vectors import DIMENSION, INDEX_NORM_TOLERANCE, coerce_index_vector

_MAGIC = b"RCFLATIX"
_VERSION = 1
_HEADER = struct.Struct("<8sIIQQI")  # magic, version, dim, count, payload_len, crc32 (index.py:40-42)

MODE_AUTO = _lib.PR_SEARCH_AUTO
MODE_EXACT = _lib.PR_SEARCH_EXACT
MODE_TENSOR = _lib.PR_SEARCH_TENSOR
MODE_TENSOR_I8 = _lib.PR_SEARCH_TENSOR_I8


@dataclass(frozen=True)
class SearchHit:
    entry_id: str
    score: float
    rank: int


def first_occurrences(rows: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """Ascending positions of the first occurrence of each value in ``rows`` (values
    in [0, pos.size)); ``pos`` is caller-owned int32 scratch, no clearing needed:
    O(len(rows)) instead of a sort."""
    n = rows.size
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    ar = np.arange(n, dtype=np.int32)
    pos[rows] = n
    np.minimum.at(pos, rows, ar)  # unbuffered: every repeat is applied (plain fancy assignment has no order guarantee)
    return np.flatnonzero(pos[rows] == ar)


# payload slot of a row whose payload is "the payload of row r of another index",
# resolved on first read (AKM rows settled device-to-device from knowledge-base rows)
_DEFERRED = object()


@dataclass
class BatchResult:
    """Device tensors of one batched search."""

    rows: Any      # int64 [B, k], -1 past count
    scores: Any    # float64 [B, k]  reported score (snap + clamp)
    raw: Any       # float64 [B, k]  einsum score
    count: Any     # int32 [B]


def _torch():
    import torch

    return torch


class FlatIndex:
    """Exact cosine k-NN over unit vectors, stored and scanned on the GPU."""

    def __init__(self, dim: int = DIMENSION, *, capacity: int = 0):
        if dim < 1:
            raise ValueError("dim must be >= 1")
        _lib.require_device()
        self._L = _lib.load()
        self._dim = dim
        self._lock = threading.RLock()
        h = ctypes.c_void_p()
        _lib.check(self._L.pr_index_create(dim, max(0, int(capacity)), 0, ctypes.byref(h)), "pr_index_create")
        self._h = h
        self._ids: list[str] = []
        self._row_by_id: dict[str, int] = {}
        self._payloads: list[Any] = []
        # deferred payload segments: (first row, source index, source rows), ascending
        self._deferred: list[tuple[int, "FlatIndex", np.ndarray]] = []
        # indices holding deferred payloads that point at rows of THIS index: pinned to the
        # current payload objects before any of this index's payloads change (upsert, clear,
        # truncate), so they keep the payload they had when copied (AKM settle semantics)
        self._dependents: "weakref.WeakSet[FlatIndex]" = weakref.WeakSet()
        self.epoch = 0  # bumped whenever rows are removed (clear / truncate)
        self.search_count = 0
        self.last_stats: _lib.SearchStats | None = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._L.pr_index_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass
            self._h = None

    # -- introspection -----------------------------------------------------
    @property
    def dim(self) -> int:
        return self._dim

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def __len__(self) -> int:
        with self._lock:
            return len(self._ids)

    def __contains__(self, entry_id: str) -> bool:
        with self._lock:
            return entry_id in self._row_by_id

    def entry_ids(self) -> tuple[str, ...]:
        with self._lock:
            return tuple(self._ids)

    def row_of(self, entry_id: str) -> int:
        with self._lock:
            return self._row_by_id[entry_id]

    def id_at(self, row: int) -> str:
        return self._ids[row]

    def payload(self, entry_id: str) -> Any:
        with self._lock:
            return self.payload_at(self._row_by_id[entry_id])

    def _pin_deferred_from(self, src: "FlatIndex") -> None:
        """Resolve every deferred payload that points at ``src`` now (``src`` is about to
        change its payloads)."""
        with self._lock:
            keep = []
            for i, (base, s_idx, rows) in enumerate(self._deferred):
                if s_idx is not src:
                    keep.append((base, s_idx, rows))
                    continue
                for j, r in enumerate(rows.tolist()):
                    if self._payloads[base + j] is _DEFERRED:
                        self._payloads[base + j] = src.payload_at(r)
            self._deferred = keep

    def _release_dependents(self) -> None:
        deps = list(self._dependents)
        self._dependents = weakref.WeakSet()
        for d in deps:
            d._pin_deferred_from(self)

    def payload_at(self, row: int) -> Any:
        p = self._payloads[row]
        if p is _DEFERRED:  # payload copied by reference from another index's row
            seg = self._deferred[bisect.bisect_right(self._deferred, row, key=lambda t: t[0]) - 1]
            p = seg[1].payload_at(int(seg[2][row - seg[0]]))
            self._payloads[row] = p
        return p

    def vector(self, entry_id: str) -> np.ndarray:
        with self._lock:
            row = self._row_by_id[entry_id]
            return self.read_rows(row, 1).cpu().numpy()[0]

    def read_rows(self, row0: int, n: int):
        torch = _torch()
        out = torch.empty((n, self._dim), dtype=torch.float32, device="cuda")
        _lib.check(self._L.pr_index_read_rows(self._h, row0, n, _lib.ptr(out), _lib.stream_ptr()), "read_rows")
        return out

    # -- writes --------------------------------------------------------------
    def insert(self, entry_id: str, vector, payload: Any = None) -> None:
        """Upsert: a new id appends a row, an existing id is overwritten in
        place and keeps its tie-break slot (index.py:125-145)."""
        arr = coerce_index_vector(vector, self._dim)
        with self._lock:
            row = self._row_by_id.get(entry_id)
            if row is None:
                self._append_rows(arr[None, :])
                self._row_by_id[entry_id] = len(self._ids)
                self._ids.append(entry_id)
                self._payloads.append(payload)
            else:
                self._release_dependents()
                self._payloads[row] = payload
                self._update_rows(np.array([row], dtype=np.int64), arr[None, :])

    def extend(self, items: Iterable[tuple[str, Any, Any]]) -> int:
        """Bulk upsert of (entry_id, vector, payload) with sequential semantics,
        shipped to the device in one append + one in-place update."""
        items = list(items)
        arrs = [coerce_index_vector(v, self._dim) for _, v, _ in items]
        with self._lock:
            new_vecs: list[np.ndarray] = []
            upd: dict[int, np.ndarray] = {}
            base = len(self._ids)
            for (eid, _, payload), arr in zip(items, arrs):
                row = self._row_by_id.get(eid)
                if row is None:
                    row = len(self._ids)
                    self._row_by_id[eid] = row
                    self._ids.append(eid)
                    self._payloads.append(payload)
                    new_vecs.append(arr)
                else:
                    if row < base:
                        self._release_dependents()
                    self._payloads[row] = payload
                    if row >= base:
                        new_vecs[row - base] = arr
                    else:
                        upd[row] = arr
            if new_vecs:
                self._append_rows(np.stack(new_vecs))
            if upd:
                rows = np.fromiter(upd.keys(), dtype=np.int64, count=len(upd))
                self._update_rows(rows, np.stack(list(upd.values())))
        return len(items)

    def extend_arrays(self, ids: list[str], vectors, payloads: list[Any] | None = None,
                      *, validate: bool = True) -> int:
        """Bulk append of NEW ids from a [n, dim] float32 array/tensor (the
        loader path: one H2D copy, device-side unit-norm validation)."""
        torch = _torch()
        t = torch.as_tensor(vectors, dtype=torch.float32)
        if t.dim() != 2 or t.shape[1] != self._dim or t.shape[0] != len(ids):
            raise InvalidVector(f"expected [{len(ids)}, {self._dim}] vectors, got {tuple(t.shape)}")
        t = t.to("cuda", non_blocking=True).contiguous()
        if validate:
            check_unit(t, INDEX_NORM_TOLERANCE)
        with self._lock:
            if any(map(self._row_by_id.__contains__, ids)):
                eid = next(e for e in ids if e in self._row_by_id)
                raise ValueError(f"extend_arrays only appends new ids; {eid!r} exists")
            base = len(self._ids)
            _lib.check(self._L.pr_index_append(self._h, _lib.ptr(t), t.shape[0], _lib.stream_ptr()), "append")
            self._row_by_id.update(zip(ids, range(base, base + len(ids))))
            self._ids.extend(ids)
            self._payloads.extend(payloads if payloads is not None else [None] * len(ids))
        return len(ids)

    def append_anonymous_from(self, src: "FlatIndex", src_rows) -> None:
        """Append rows copied from ``src`` without ids or payloads (scratch stores that
        are only searched, never looked up by id)."""
        torch = _torch()
        r = _lib.h2d(src_rows, torch.int64)
        with self._lock:
            self._copy_rows_from(src, r)
            self._ids.extend([None] * r.numel())
            self._payloads.extend([None] * r.numel())

    def append_rows_from(self, src: "FlatIndex", src_rows, ids: list[str], payloads: list[Any] | None = None) -> None:
        """Append rows copied device-to-device from another index (AKM settle
        from knowledge-base rows).  ``payloads=None``: each new row's payload is
        the source row's, read from ``src`` on first access."""
        torch = _torch()
        rows = np.asarray(src_rows, dtype=np.int64)
        r = _lib.h2d(rows)
        with self._lock:
            base = len(self._ids)
            self._copy_rows_from(src, r)
            self._row_by_id.update(zip(ids, range(base, base + len(ids))))
            self._ids.extend(ids)
            if payloads is None:
                self._deferred.append((base, src, rows))
                src._dependents.add(self)
                self._payloads.extend([_DEFERRED] * len(ids))
            else:
                self._payloads.extend(payloads)

    def _copy_rows_from(self, src: "FlatIndex", r) -> None:
        """Append the device rows ``r`` (int64 device tensor) of ``src``: device to device,
        or for a row-sharded source (sharded.ShardedRowIndex) its exact fp32 rows gathered
        from their owning ranks."""
        if getattr(src, "sharded", False):
            v = src.gather_vectors(r)
            _lib.check(self._L.pr_index_append(self._h, _lib.ptr(v), v.shape[0], _lib.stream_ptr()), "append")
            return
        _lib.check(self._L.pr_index_append_from(self._h, src.handle, _lib.ptr(r), r.numel(), _lib.stream_ptr()),
                   "append_from")

    def _append_rows(self, arr: np.ndarray) -> None:
        torch = _torch()
        t = torch.from_numpy(np.require(arr, np.float32, ["C", "W"])).to("cuda", non_blocking=False)
        _lib.check(self._L.pr_index_append(self._h, _lib.ptr(t), t.shape[0], _lib.stream_ptr()), "append")

    def _update_rows(self, rows: np.ndarray, arr: np.ndarray) -> None:
        torch = _torch()
        r = torch.from_numpy(rows).to("cuda")
        t = torch.from_numpy(np.require(arr, np.float32, ["C", "W"])).to("cuda")
        _lib.check(self._L.pr_index_update_rows(self._h, _lib.ptr(r), _lib.ptr(t), t.shape[0], _lib.stream_ptr()),
                   "update")

    def clear(self) -> None:
        with self._lock:
            self._release_dependents()
            self._ids.clear()
            self._row_by_id.clear()
            self._payloads.clear()
            self._deferred.clear()
            self.epoch += 1
            _lib.check(self._L.pr_index_clear(self._h), "clear")

    def truncate(self, n: int) -> None:
        with self._lock:
            if n < len(self._ids):
                self._release_dependents()
            for eid in self._ids[n:]:
                del self._row_by_id[eid]
            del self._ids[n:]
            del self._payloads[n:]
            while self._deferred and self._deferred[-1][0] >= n:
                self._deferred.pop()
            self.epoch += 1
            _lib.check(self._L.pr_index_truncate(self._h, n), "truncate")

    # -- search ----------------------------------------------------------------
    def search_batch(self, queries, k: int, *, mode: int = MODE_AUTO, validate: bool = True,
                     out: BatchResult | None = None, row_limit=None, count: bool = True,
                     floor: float | None = None) -> BatchResult:
        """Batched FlatIndex.search.  ``queries``: [B, dim] float32 (torch
        tensor on any device, or numpy).  Returns device tensors; counts
        ``search_count`` once per query like B sequential calls (unless
        ``count=False``).  ``row_limit`` (int64 [B]) restricts query b to rows
        [0, row_limit[b]) — the store as it was earlier in a sequential stream.
        ``floor``: the caller only acts on scores >= floor (a cache threshold):
        results at or above it are exact, rows below it may be missing
        (``pr_index_search_floor``) — ``count > 0 and scores[:, 0] >= floor``
        is then exactly the full search's threshold decision."""
        if k < 1:
            raise ValueError("k must be >= 1")
        torch = _torch()
        if isinstance(queries, np.ndarray) and not queries.flags.writeable:
            queries = np.array(queries)  # torch refuses read-only numpy memory (EmbeddingVector values)
        q = torch.as_tensor(queries, dtype=torch.float32)
        if q.dim() != 2 or q.shape[1] != self._dim:
            raise InvalidVector(f"expected [B, {self._dim}] queries, got {tuple(q.shape)}")
        q = _lib.h2d(q).contiguous()
        B = q.shape[0]
        if validate and B:
            check_unit(q, INDEX_NORM_TOLERANCE)
        if out is None:
            out = BatchResult(
                rows=torch.empty((B, k), dtype=torch.int64, device="cuda"),
                scores=torch.empty((B, k), dtype=torch.float64, device="cuda"),
                raw=torch.empty((B, k), dtype=torch.float64, device="cuda"),
                count=torch.empty((B,), dtype=torch.int32, device="cuda"),
            )
        lim = None
        if row_limit is not None:
            lim = _lib.h2d(row_limit, torch.int64).contiguous()
            if lim.shape != (B,):
                raise ValueError("row_limit must have one entry per query")
        with self._lock:
            if count:
                self.search_count += B
            if B:
                if floor is None:
                    rc = self._L.pr_index_search_ex(
                        self._h, _lib.ptr(q), B, k, mode, _lib.ptr(lim), _lib.ptr(out.rows), _lib.ptr(out.raw),
                        _lib.ptr(out.scores), _lib.ptr(out.count), _lib.stream_ptr(),
                    )
                else:
                    rc = self._L.pr_index_search_floor(
                        self._h, _lib.ptr(q), B, k, mode, _lib.ptr(lim), float(floor), _lib.ptr(out.rows),
                        _lib.ptr(out.raw), _lib.ptr(out.scores), _lib.ptr(out.count), _lib.stream_ptr(),
                    )
                _lib.check(rc, "pr_index_search")
        return out

    def set_timing(self, enable: bool = True) -> None:
        """Record CUDA events around the dominant scan kernel of every search."""
        _lib.check(self._L.pr_index_set_timing(self._h, 1 if enable else 0), "set_timing")

    def scan_time(self) -> tuple[float, int]:
        """(summed kernel ms, launches) since the last call; synchronises."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        _lib.check(self._L.pr_index_scan_time(self._h, ctypes.byref(ms), ctypes.byref(n)), "scan_time")
        return ms.value, n.value

    def stats(self) -> _lib.SearchStats:
        st = _lib.SearchStats()
        _lib.check(self._L.pr_index_last_stats(self._h, ctypes.byref(st)), "last_stats")
        return st

    def search(self, query_vector, k: int, *, mode: int = MODE_AUTO) -> list[SearchHit]:
        """Exact top-k by cosine, ties by insertion order (index.py:155-189)."""
        if k < 1:
            raise ValueError("k must be >= 1")
        q32 = coerce_index_vector(query_vector, self._dim)
        with self._lock:
            res = self.search_batch(q32[None, :], k, mode=mode, validate=False)
            n = int(res.count[0].item())
            rows = res.rows[0, :n].cpu().numpy()
            scores = res.scores[0, :n].cpu().numpy()
            return [SearchHit(self._ids[int(r)], float(s), i + 1) for i, (r, s) in enumerate(zip(rows, scores))]

    def hits_from_batch(self, res: BatchResult) -> list[list[SearchHit]]:
        counts = res.count.cpu().numpy()
        rows = res.rows.cpu().numpy()
        scores = res.scores.cpu().numpy()
        out = []
        for b in range(rows.shape[0]):
            out.append([SearchHit(self._ids[int(rows[b, j])], float(scores[b, j]), j + 1) for j in range(counts[b])])
        return out

    # -- snapshot / restore (index.py:198-261) ----------------------------
    def snapshot(self, payload_encoder: Callable[[Any], Any] | None = None) -> bytes:
        enc = payload_encoder or (lambda p: p)
        with self._lock:
            n = len(self._ids)
            vec_block = self.read_rows(0, n).cpu().numpy().tobytes() if n else b""
            lines = [json.dumps({"id": self._ids[i], "payload": enc(self.payload_at(i))}, ensure_ascii=False)
                     for i in range(n)]
            meta = ("\n".join(lines) + ("\n" if lines else "")).encode("utf-8")
            body = vec_block + meta
            return _HEADER.pack(_MAGIC, _VERSION, self._dim, n, len(meta), zlib.crc32(body)) + body

    @classmethod
    def restore(cls, data: bytes, payload_decoder: Callable[[Any], Any] | None = None) -> "FlatIndex":
        """FlatIndex.restore (index.py:222-261) as a bulk device load: the
        vector block goes to HBM in one pinned H2D copy and is appended in one call,
        instead of one validated insert per record.  Same result as the reference's
        per-record ``insert`` loop: a repeated id keeps the row of its first record and
        takes the vector and payload of its last; any non-unit vector raises
        InvalidVector."""
        torch = _torch()
        dec = payload_decoder or (lambda p: p)
        dim, vecs, recs = parse_snapshot(data)
        first: dict[str, int] = {}
        last: dict[str, int] = {}
        for i, r in enumerate(recs):
            first.setdefault(r["id"], i)
            last[r["id"]] = i
        order = list(first)
        idx = cls(dim=dim, capacity=max(1, len(order)))
        if not order:
            return idx
        host = torch.from_numpy(np.array(vecs, copy=True)).pin_memory()
        block = host.to("cuda", non_blocking=True)
        check_unit(block, INDEX_NORM_TOLERANCE)  # every record is validated, as each insert would be
        src = torch.as_tensor(np.fromiter((last[e] for e in order), dtype=np.int64, count=len(order))).cuda()
        idx.extend_arrays(order, block.index_select(0, src), [dec(recs[last[e]].get("payload")) for e in order],
                          validate=False)
        return idx


def parse_snapshot(data: bytes) -> tuple[int, np.ndarray, list[dict]]:
    """Host half of restore: header, length and crc checks, the fp32 block (a view of
    ``data``) and the JSON sidecar, with the reference's CorruptSnapshot cases
    (index.py:234-258)."""
    if len(data) < _HEADER.size:
        raise CorruptSnapshot("snapshot shorter than header")
    magic, version, dim, count, meta_len, crc = _HEADER.unpack_from(data)
    if magic != _MAGIC:
        raise CorruptSnapshot(f"bad magic {magic!r}")
    if version != _VERSION:
        raise CorruptSnapshot(f"unsupported snapshot version {version}")
    body = memoryview(data)[_HEADER.size:]
    vec_len = count * dim * 4
    if len(body) != vec_len + meta_len:
        raise CorruptSnapshot(f"body length {len(body)} != expected {vec_len + meta_len}")
    if zlib.crc32(body) != crc:
        raise CorruptSnapshot("checksum mismatch")
    vecs = np.frombuffer(body[:vec_len], dtype=np.float32).reshape(count, dim)
    meta = bytes(body[vec_len:]).decode("utf-8").splitlines()
    if len(meta) != count:
        raise CorruptSnapshot(f"payload sidecar has {len(meta)} lines, expected {count}")
    recs = []
    for i, line in enumerate(meta):
        try:
            recs.append(json.loads(line))
        except json.JSONDecodeError as exc:
            raise CorruptSnapshot(f"payload line {i + 1}: {exc}") from exc
    return dim, vecs, recs


def check_unit(t, tol: float) -> None:
    """Device-side unit-norm/finiteness check of a [n, dim] float32 CUDA tensor."""
    torch = _torch()
    L = _lib.load()
    bad = torch.empty((t.shape[0],), dtype=torch.uint8, device="cuda")
    _lib.check(L.pr_check_unit(_lib.ptr(t), t.shape[0], t.shape[1], tol, _lib.ptr(bad), _lib.stream_ptr()),
               "check_unit")
    if bool(bad.any().item()):
        i = int(torch.nonzero(bad)[0].item())
        raise InvalidVector(f"vector {i} is not finite unit-norm within {tol}")
