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

from dataclasses import dataclass
from typing import Callable

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
