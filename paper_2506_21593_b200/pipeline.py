"""Streaming batched search from host memory: the serving loop of a retrieval front end.

``search_stream(index, host_batches, k)`` searches a sequence of query batches that live in
(pinned) host memory and yields each batch's results in host memory, in order — exactly
``[index.search_batch(b, k) for b in host_batches]`` copied back to the host — with the
transfers overlapped with the scans: batch i+1's host→device copy and batch i−1's
device→host copy run on a copy stream while batch i is scanned.  Query and result buffers
are double-buffered on the device and in pinned host memory, and every cross-stream use is
ordered by CUDA events, so no buffer is overwritten before its consumer finished.

``index`` is a ``FlatIndex`` or a ``ShardedFlatIndex`` (one all-gather per batch on more
than one rank: the collective runs on the compute stream, as in ``search_batch``).
"""
from __future__ import annotations

from typing import Iterable, Iterator

from .index import MODE_AUTO, BatchResult, FlatIndex


def search_stream(index, host_batches: Iterable, k: int, *, mode: int = MODE_AUTO) -> Iterator[tuple]:
    """Yield (rows int64 [B, k], scores float64 [B, k], count int32 [B]) host tensors per
    batch (pinned buffers, reused: a triple is valid until the generator advances)."""
    import torch

    local = getattr(index, "local", None)
    flat = index if isinstance(index, FlatIndex) else (
        local if local is not None and getattr(index, "world", 1) == 1 else None)
    main = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    dq: list = [None, None]
    dres: list = [None, None]
    hres: list = [None, None]
    ev_h2d = [torch.cuda.Event(), torch.cuda.Event()]
    ev_scan = [torch.cuda.Event(), torch.cuda.Event()]
    ev_d2h = [torch.cuda.Event(), torch.cuda.Event()]
    scanned = [False, False]

    def upload(i, hb):
        s = i & 1
        if dq[s] is None or dq[s].shape != hb.shape:
            dq[s] = torch.empty(hb.shape, dtype=torch.float32, device="cuda")
        with torch.cuda.stream(copy):
            if scanned[s]:
                copy.wait_event(ev_scan[s])  # the scan that read this buffer two batches ago
            dq[s].copy_(hb, non_blocking=True)
            ev_h2d[s].record(copy)

    def scan(i, B):
        s = i & 1
        main.wait_event(ev_h2d[s])
        if flat is not None:
            r = dres[s]
            if r is None or r.rows.shape != (B, k):
                r = dres[s] = BatchResult(
                    rows=torch.empty((B, k), dtype=torch.int64, device="cuda"),
                    scores=torch.empty((B, k), dtype=torch.float64, device="cuda"),
                    raw=torch.empty((B, k), dtype=torch.float64, device="cuda"),
                    count=torch.empty((B,), dtype=torch.int32, device="cuda"))
            else:
                main.wait_event(ev_d2h[s])  # the previous results in this buffer reached the host
            flat.search_batch(dq[s], k, mode=mode, validate=False, out=r)
        else:
            r = dres[s] = index.search_batch(dq[s], k, mode=mode)
            for t in (r.rows, r.scores, r.count):
                t.record_stream(copy)
        ev_scan[s].record(main)
        scanned[s] = True

    def download(i, B):
        s = i & 1
        h = hres[s]
        if h is None or h[0].shape != (B, k):
            h = hres[s] = (torch.empty((B, k), dtype=torch.int64).pin_memory(),
                           torch.empty((B, k), dtype=torch.float64).pin_memory(),
                           torch.empty((B,), dtype=torch.int32).pin_memory())
        r = dres[s]
        with torch.cuda.stream(copy):
            copy.wait_event(ev_scan[s])
            h[0].copy_(r.rows, non_blocking=True)
            h[1].copy_(r.scores, non_blocking=True)
            h[2].copy_(r.count, non_blocking=True)
            ev_d2h[s].record(copy)

    it = iter(host_batches)
    cur = next(it, None)
    if cur is None:
        return
    try:
        i = 0
        upload(0, cur)
        pending = None  # index of the batch whose results are on their way to the host
        while cur is not None:
            nxt = next(it, None)
            scan(i, cur.shape[0])
            if nxt is not None:
                upload(i + 1, nxt)  # overlaps scan i
            download(i, cur.shape[0])  # overlaps scan i + 1
            if pending is not None:
                ev_d2h[pending & 1].synchronize()
                yield hres[pending & 1]
            pending = i
            cur = nxt
            i += 1
        ev_d2h[pending & 1].synchronize()
        yield hres[pending & 1]
    finally:
        # a consumer that stops early (or an exception) must not free buffers the copy
        # stream still reads or writes
        copy.synchronize()
