"""Row-sharded flat index across ranks (one process per GPU).

The store is split into contiguous row blocks — rank r holds global rows
[offset_r, offset_r + n_r) — so global row order is still insertion order and
the reference's (score desc, row asc) tie-break (index.py:176) survives the
split.  A batched search runs the local exact top-k on every rank, tags each
hit with its global row and the rank-local self-snap predicate
(index.py:180-181, which needs the stored row), exchanges the per-rank lists
with ONE all-gather (NCCL over NVLink on the GPU box, gloo in the CPU tests),
and merges them on the device (pr_merge_shards).  The merge is exact: every
global top-k hit is in its own rank's local top-k.

The local search and the merge are injectable so the distributed plumbing
can be exercised on CPU with gloo; in production both are libpentarag calls.
"""
from __future__ import annotations

import threading
import weakref
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib
from .index import MODE_AUTO, BatchResult, FlatIndex


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row block of rank ``rank`` (first n % world ranks get one more)."""
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


@dataclass
class LocalHits:
    rows: object    # int64 [B, k] GLOBAL row ids, -1 past count
    raw: object     # float64 [B, k]
    snap: object    # uint8 [B, k]
    count: object   # int32 [B]


def pack(h: LocalHits):
    """One int64 buffer per rank: rows | raw bits | snap | count."""
    import torch

    B, k = h.rows.shape
    return torch.cat([
        h.rows.reshape(-1),
        h.raw.contiguous().view(torch.int64).reshape(-1),
        h.snap.to(torch.int64).reshape(-1),
        h.count.to(torch.int64).reshape(-1),
    ])


def unpack(buf, B: int, k: int) -> LocalHits:
    import torch

    n = B * k
    rows = buf[:n].view(B, k)
    raw = buf[n:2 * n].clone().view(torch.float64).view(B, k)
    snap = buf[2 * n:3 * n].to(torch.uint8).view(B, k)
    count = buf[3 * n:3 * n + B].to(torch.int32)
    return LocalHits(rows, raw, snap, count)


class ShardedFlatIndex:
    """A rank's shard plus the all-gather merge."""

    def __init__(self, local: FlatIndex | None, row_offset: int, *, group=None,
                 local_search: Callable | None = None, merge: Callable | None = None):
        import torch.distributed as dist

        self.local = local
        self.row_offset = int(row_offset)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self._local_search = local_search or self._device_local_search
        self._merge = merge or device_merge

    # production path -------------------------------------------------------
    def _device_local_search(self, q, k: int, mode: int) -> LocalHits:
        import torch

        res = self.local.search_batch(q, k, mode=mode, validate=False)
        B = q.shape[0]
        snap = torch.empty((B, k), dtype=torch.uint8, device=q.device)
        L = _lib.load()
        _lib.check(L.pr_index_snap_flags(self.local.handle, _lib.ptr(q), B, k, _lib.ptr(res.rows),
                                         _lib.ptr(res.raw), _lib.ptr(res.count), 0, _lib.ptr(snap),
                                         _lib.stream_ptr()), "snap_flags")
        rows = torch.where(res.rows >= 0, res.rows + self.row_offset, res.rows)
        return LocalHits(rows, res.raw, snap, res.count)

    def search_batch(self, q, k: int, *, mode: int = MODE_AUTO) -> BatchResult:
        import torch.distributed as dist

        B = q.shape[0]
        if self.world == 1 and self.local is not None and self._merge is device_merge:
            # single shard: the local exact top-k already is the answer
            return self.local.search_batch(q, k, mode=mode, validate=False)
        mine = self._local_search(q, k, mode)
        if self.world == 1:
            parts = [mine]
        else:
            buf = pack(mine)
            bufs = [buf.new_empty(buf.shape) for _ in range(self.world)]
            dist.all_gather(bufs, buf, group=self.group)
            parts = [unpack(b, B, k) for b in bufs]
        return self._merge(parts, B, k)


def device_merge(parts: list[LocalHits], B: int, k: int) -> BatchResult:
    import torch

    rows = torch.stack([p.rows for p in parts]).contiguous()
    raw = torch.stack([p.raw for p in parts]).contiguous()
    snap = torch.stack([p.snap for p in parts]).contiguous()
    count = torch.stack([p.count for p in parts]).contiguous()
    dev = rows.device
    out = BatchResult(
        rows=torch.empty((B, k), dtype=torch.int64, device=dev),
        scores=torch.empty((B, k), dtype=torch.float64, device=dev),
        raw=torch.empty((B, k), dtype=torch.float64, device=dev),
        count=torch.empty((B,), dtype=torch.int32, device=dev),
    )
    L = _lib.load()
    _lib.check(L.pr_merge_shards(_lib.ptr(rows), _lib.ptr(raw), _lib.ptr(snap), _lib.ptr(count), len(parts), B, k,
                                 _lib.ptr(out.rows), _lib.ptr(out.raw), _lib.ptr(out.scores), _lib.ptr(out.count),
                                 _lib.stream_ptr()), "merge_shards")
    return out


class _LocalView(FlatIndex):
    """A FlatIndex sharing another index's device handle (never destroys it)."""

    def __del__(self):
        pass


class ShardedRowIndex(FlatIndex):
    """A ``FlatIndex`` drop-in whose device rows are row-sharded over the ranks of a process
    group (the knowledge base of a multi-GPU cascade): rank r's device store
    holds the contiguous global block ``shard_range(n, r, world)``, while the host side —
    ids, payloads, counters — covers every row on every rank, so the router's host logic
    (answers, AKM ids, write-back bookkeeping) runs unchanged and identically on all ranks.

    * ``search_batch`` / ``search_list``: local exact top-k on the shard, per-rank self-snap
      flags, ONE all-gather of B·(3k+1) int64, device merge (``pr_merge_shards``) — the
      unsharded answer bit for bit (contiguous blocks keep global row order).
    * ``gather_vectors``: exact fp32 rows of arbitrary global rows (owners copy, the rest
      zero, one SUM all-reduce of the int32 bit patterns) — how the AKM settle and the
      cascade's seed guard copy knowledge-base rows that live on other ranks.

    Every rank must make the same calls in the same order (the cascade is deterministic and
    replicated, so it does).  The store is loaded once (``load``); upserts / truncation are
    not supported."""

    sharded = True

    def __init__(self, dim: int, *, group=None):
        import torch.distributed as dist

        super().__init__(dim=dim)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.row_offset = 0
        self.n_local = 0

    @classmethod
    def load(cls, ids: list[str], payloads: list, local_vectors, *, dim: int, group=None,
             validate: bool = True) -> "ShardedRowIndex":
        """``ids`` / ``payloads``: every global row (same on all ranks); ``local_vectors``:
        this rank's block ``shard_range(len(ids), rank, world)`` as a [n_r, dim] array."""
        self = cls(dim, group=group)
        lo, hi = shard_range(len(ids), self.rank, self.world)
        t = _lib.h2d(local_vectors).float().contiguous() if local_vectors is not None else None
        if t is None or t.shape != (hi - lo, dim):
            raise ValueError(f"rank {self.rank}: expected local rows [{lo}, {hi}) x {dim}")
        self.local_store().extend_arrays([str(i) for i in range(lo, hi)], t, validate=validate)
        self.row_offset, self.n_local = lo, hi - lo
        self._ids = list(ids)
        self._row_by_id = {e: i for i, e in enumerate(ids)}
        self._payloads = list(payloads)
        return self

    @classmethod
    def wrap(cls, local: FlatIndex, ids: list[str], payloads, row_offset: int, *, group=None) -> "ShardedRowIndex":
        """A sharded view over an already loaded local block (``local`` holds global rows
        [row_offset, row_offset + len(local))); ``ids`` / ``payloads`` cover every row."""
        import torch.distributed as dist

        self = cls.__new__(cls)
        self._L, self._dim, self._h = local._L, local._dim, local._h
        self._lock = threading.RLock()
        self._owner, self._owns_handle = local, False
        self._ids = list(ids)
        self._row_by_id = {e: i for i, e in enumerate(self._ids)}
        self._payloads = payloads
        self._deferred, self._dependents = [], weakref.WeakSet()
        self.epoch = self.search_count = 0
        self.last_stats = None
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.row_offset, self.n_local = int(row_offset), len(local)
        return self

    def local_store(self) -> FlatIndex:
        """This rank's device rows as a plain FlatIndex view (the handle is shared)."""
        v = _LocalView.__new__(_LocalView)
        v.__dict__.update({k: getattr(self, k) for k in ("_L", "_dim", "_h", "_lock")})
        v._ids, v._row_by_id, v._payloads, v._deferred = [], {}, [], []
        v._dependents = weakref.WeakSet()
        v.epoch = v.search_count = 0
        v.last_stats = None
        v._view_of = self  # keeps the owner (and its handle) alive
        return v

    def __del__(self):
        if getattr(self, "_owns_handle", True):
            FlatIndex.__del__(self)

    # -- collectives -----------------------------------------------------------
    def _all_gather(self, buf):
        import torch.distributed as dist

        if self.world == 1:
            return [buf]
        bufs = [buf.new_empty(buf.shape) for _ in range(self.world)]
        dist.all_gather(bufs, buf, group=self.group)
        return bufs

    def gather_vectors(self, rows):
        """[m, dim] float32 device tensor of the global rows ``rows`` (device int64)."""
        import torch
        import torch.distributed as dist

        rows = _lib.h2d(rows, torch.int64).contiguous()
        out = torch.empty((rows.numel(), self._dim), dtype=torch.float32, device="cuda")
        if rows.numel():
            _lib.check(self._L.pr_index_gather_rows(self._h, _lib.ptr(rows), rows.numel(), self.row_offset,
                                                    _lib.ptr(out), _lib.stream_ptr()), "gather_rows")
        if self.world > 1:
            iv = out.view(torch.int32)
            dist.all_reduce(iv, op=dist.ReduceOp.SUM, group=self.group)
        return out

    def _merge_local(self, q, k, rows, raw, count) -> BatchResult:
        import torch

        B = q.shape[0]
        snap = torch.empty((B, k), dtype=torch.uint8, device="cuda")
        _lib.check(self._L.pr_index_snap_flags(self._h, _lib.ptr(q), B, k, _lib.ptr(rows), _lib.ptr(raw),
                                               _lib.ptr(count), 0, _lib.ptr(snap), _lib.stream_ptr()), "snap_flags")
        g = torch.where(rows >= 0, rows + self.row_offset, rows)
        mine = LocalHits(g, raw, snap, count)
        if self.world == 1:
            parts = [mine]
        else:
            parts = [unpack(b, B, k) for b in self._all_gather(pack(mine))]
        return device_merge(parts, B, k)

    # -- search ----------------------------------------------------------------
    def search_batch(self, queries, k: int, *, mode: int = MODE_AUTO, validate: bool = True,
                     out: BatchResult | None = None, row_limit=None, count: bool = True) -> BatchResult:
        import torch

        q = _lib.h2d(queries.float() if isinstance(queries, torch.Tensor)
                     else np.asarray(queries, dtype=np.float32)).contiguous()
        lim = None
        if row_limit is not None:
            lim = (_lib.h2d(row_limit, torch.int64) - self.row_offset).clamp(0, self.n_local).contiguous()
        local = FlatIndex.search_batch(self.local_store(), q, k, mode=mode, validate=validate, row_limit=lim,
                                       count=False)
        res = self._merge_local(q, k, local.rows, local.raw, local.count)
        if count:
            with self._lock:
                self.search_count += q.shape[0]
        if out is not None:
            for f in ("rows", "scores", "raw", "count"):
                getattr(out, f).copy_(getattr(res, f))
            return out
        return res

    def search_list(self, Vd, lst, nlist, B: int, hint: int, k: int, mode: int, rows, raw, rep, cnt) -> None:
        """pr_index_search_list over the shard + all-gather merge; outputs per listed position
        (positions >= *nlist report count 0), global rows."""
        import torch

        lrows = torch.empty((B, k), dtype=torch.int64, device="cuda")
        lraw = torch.empty((B, k), dtype=torch.float64, device="cuda")
        lrep = torch.empty((B, k), dtype=torch.float64, device="cuda")
        lcnt = torch.empty(B, dtype=torch.int32, device="cuda")
        with self._lock:
            _lib.check(self._L.pr_index_search_list(self._h, _lib.ptr(Vd), _lib.ptr(lst), _lib.ptr(nlist), B, hint, k,
                                                    mode, None, _lib.ptr(lrows), _lib.ptr(lraw), _lib.ptr(lrep),
                                                    _lib.ptr(lcnt), _lib.stream_ptr()), "search_list")
        live = torch.arange(B, device="cuda") < nlist.to(torch.int64)
        lcnt = torch.where(live, lcnt, torch.zeros_like(lcnt))
        lrows = torch.where(live[:, None], lrows, torch.full_like(lrows, -1))
        lraw = torch.where(live[:, None], lraw, torch.zeros_like(lraw))
        qc = Vd.index_select(0, lst.long().clamp(0, max(0, Vd.shape[0] - 1))).contiguous()
        res = self._merge_local(qc, k, lrows, lraw, lcnt)
        rows.copy_(res.rows)
        raw.copy_(res.raw)
        rep.copy_(res.scores)
        cnt.copy_(res.count)

    def read_rows(self, row0: int, n: int):
        import torch

        return self.gather_vectors(torch.arange(row0, row0 + n, dtype=torch.int64, device="cuda"))

    # -- the store is loaded once ------------------------------------------------
    def _unsupported(self, *a, **kw):
        raise NotImplementedError("ShardedRowIndex is loaded once (ShardedRowIndex.load); no in-place edits")

    insert = extend = extend_arrays = append_anonymous_from = append_rows_from = _unsupported
    _append_rows = _update_rows = clear = truncate = _unsupported

    @property
    def handle(self):
        raise AttributeError("a ShardedRowIndex has no single device handle: use search_list / gather_vectors")
