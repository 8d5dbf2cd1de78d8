"""Batched, sequential-equivalent routing with the cascade on the device.

``route_batch(router, queries)`` returns exactly what ``[router.route(q) for q in queries]``
returns — answers, trace events, store contents and every counter.  The queries are cut
into spans (``span`` queries, 4096 by default) and every span runs in two stages:

DEVICE stage (``_launch``, enqueued on the router's CUDA stream, no host read-back):

* L1 (fixed KV, router.py:232): one fused hash + probe kernel over the span's UTF-8 arena;
  a query also hits if an EARLIER query of the span or of the previous span had the same
  text (every served answer is written back before the next query, router.py:333-337) —
  the window's first-occurrence map is host-side (texts only), uploaded as a mask.
* L2 (semantic cache, caches.py:131-145): the first occurrence of every text new to the
  cache is appended up front (that is what write-back will do), and ONE row-limited top-1
  search lets query j see exactly the rows written by queries before it.  The router only
  acts on a top-1 at or above the threshold, so the L2 and L4 searches are threshold
  searches (``floor``: exact at and above it, the int8 scan starts from it).
* L3 (memory recall, generation.py:203-224), when the backend is the stub LLM over a
  ``DeviceKnowledgeTable``: one probe of the recall hash table + the confidence gate
  (``pr_recall_gate``).  The table never changes while routing, so no window is needed.
* Gate (``pr_cascade_gate``): L1 / L2 / L3 outcomes in probe order, and the ONE compacted
  miss list — the queries no fast layer answered — built on the device by a prefix sum.
* L5 (knowledge base, knowledge.py:65-85): one top-seed_k scan of the listed queries only
  (``pr_index_search_list``: the list and its count never leave the device).
* L4 guard: L4 depends on which earlier queries were served by L5 (their seeds settle into
  the AKM before the next query, router.py:284-285), a routing OUTCOME.  The span proves L4
  misses instead: top-1 over the AKM and over a superset of every seed an earlier query
  could contribute (``pr_cascade_seeds``: seeds of the previous span's and this span's
  listed queries, deduplicated on the device; row-limited scan of a scratch store).
* The outcomes are packed and copied to pinned host memory: the span's ONE read-back.

HOST stage (``_finish``): the decision pass over the span (vectorised), answers as
columns (``ledger.BatchLedger``; objects are built lazily), write-back (KV put on the
device, semantic-cache payloads, AKM settle device-to-device from KB rows) and counters.
If the L4 guard cannot prove a miss for some query, the span stops before it, that query
is routed by ``router.route`` exactly, and batching resumes after it.

Pipelining: span i+1's device stage is enqueued BEFORE span i's host stage, so the host's
bookkeeping of span i overlaps the GPU's scans of span i+1.  This is exact because span
i+1's device stage depends on span i only through texts and vectors (L1 window mask, the
semantic-cache rows appended up front) and through span i's seeds (included in the L4 guard
superset), never through span i's answers.  If span i stops early, span i+1's speculative
results are discarded (its cache rows are rolled back) and the pipeline restarts.

All scores are the exact fp64 reference scores (bit-identical), so every threshold
decision is the reference's.  Regimes that need per-query state changes inside a span
fall back to ``route`` per query: no knowledge base / NAIVE_RAG disabled (queries may miss
every layer and skip write-back), capped caches (LRU eviction), or a non-deterministic AKM
settle thread.
"""
from __future__ import annotations

import ctypes
import os
import time
from collections import deque
from itertools import repeat
from operator import attrgetter, getitem, is_, itemgetter

import numpy as np

from . import _lib, generation, pinned
from .caches import FixedKVCache, SemanticCache
from .errors import CascadeError
from .index import _DEFERRED, MODE_AUTO, FlatIndex
from .knowledge import AdaptiveKnowledgeMemory
from .ledger import BatchLedger, CtxRows, LedgerEntry, entries_of, entry_text_conf
from .records import LayerTag
from .router import LayerProbe
from .textarena import to_device

L1, L2, L3, L4, L5 = (LayerTag.FIXED_KV, LayerTag.SEMANTIC_CACHE, LayerTag.MEMORY_RECALL,
                      LayerTag.ADAPTIVE_MEMORY, LayerTag.NAIVE_RAG)
# immutable probe records shared by every routed query (only the serving
# layer's probe carries a latency and is built per query)
_PROBE = {(L, o): LayerProbe(L, o) for L in LayerTag for o in ("hit", "miss", "rejected")}
DEFAULT_SPAN = 4096


def batchable(router) -> bool:
    cfg = router.config
    return (
        L5 in cfg.probe_order()
        and len(router.knowledge_base) > 0
        and cfg.deterministic_settle
        and isinstance(router.kv_cache, FixedKVCache) and router.kv_cache._max_entries is None
        and isinstance(router.semantic_cache, SemanticCache) and router.semantic_cache._max_entries is None
        and isinstance(router.adaptive_memory, AdaptiveKnowledgeMemory)
    )


def route_batch(router, queries, vectors=None, *, mode: int = MODE_AUTO, materialize: bool = True,
                capture_errors: bool = False, span: int = DEFAULT_SPAN):
    """Route ``queries`` in order; see the module docstring.  Returns the list
    of (AnswerRecord, RouteTraceEvent), or with ``materialize=False`` a
    ``RoutedBatch`` of columnar segments (objects built only on access).

    ``capture_errors``: a query whose ``route`` raises a CascadeError (e.g.
    AllLayersMissed, router.py:309-323 — no write-back happens for it) gets the
    exception object as its result and the batch continues, exactly like
    independent ``route`` calls would (service micro-batching)."""
    segs = []
    i, n = 0, len(queries)
    stats = {"batched": 0, "sequential": 0, "splits": 0, "spans": 0, "pipelined": 0}
    span = max(1, int(span))
    kv = router.kv_cache

    def one(q):
        if not capture_errors:
            return router.route(q)
        try:
            return router.route(q)
        except CascadeError as exc:
            return exc

    pending = None
    # KV values (write sequence numbers = arena indices) read by a launched span stay valid
    # until its host stage: no arena compaction of the fixed-KV cache, nor of a device recall
    # table (an add from another thread could otherwise compact it between probe and decision)
    held = [c for c in (kv, getattr(getattr(router.backend, "knowledge", None), "_kv", None))
            if isinstance(c, FixedKVCache)]
    for c in held:
        c._compact_hold += 1
    try:
        while i < n:
            if not batchable(router):
                pending = None
                segs.append([one(queries[i])])
                stats["sequential"] += 1
                i += 1
                continue
            if pending is not None and pending.start == i:
                cur, pending = pending, None
                stats["pipelined"] += 1
            else:
                router.adaptive_memory.settle()  # the first route() would settle the queue (router.py:284-285)
                cur = _launch(router, queries, vectors, i, min(n, i + span), mode, None)
            if cur.end < n:
                # span i+1's device work is queued before span i's host stage (module doc)
                pending = _launch(router, queries, vectors, cur.end, min(n, cur.end + span), mode, cur)
            stats["spans"] += 1
            try:
                done, ledger = _finish(router, cur, more_follow=cur.end < n)
            except _BackendFailed:
                # a backend call raised: every store mutation of the span (and of the
                # speculative next span) was rolled back — route the rest one by one, so
                # the failing query raises (or is captured) where independent route()
                # calls would raise
                pending = None
                for q in queries[i:]:
                    segs.append([one(q)])
                stats["sequential"] += n - i
                break
            if done:
                segs.append(ledger)
            stats["batched"] += done
            i += done
            if done < cur.size:
                # the next query's AKM outcome is not certain: route it exactly.  The
                # speculative next span assumed this span was served in full: drop it
                # (its cache rows went with the truncation in _writeback)
                pending = None
                segs.append([one(queries[i])])
                stats["sequential"] += 1
                stats["splits"] += 1
                i += 1
    finally:
        if pending is not None:
            _discard(router, pending)
        for c in held:
            c._compact_hold -= 1
            if not c._compact_hold:
                with c._lock:
                    c._maybe_compact()
    router.last_batch_stats = stats
    rb = RoutedBatch(segs)
    return rb.results() if materialize else rb


class RoutedBatch:
    """Concatenation of ledgers (batched spans) and (answer, event) lists (queries routed one by one)."""

    def __init__(self, segs):
        self.segs = segs

    def __len__(self) -> int:
        return sum(len(s) for s in self.segs)

    def results(self) -> list:
        out = []
        for s in self.segs:
            out.extend(s.results() if isinstance(s, BatchLedger) else s)
        return out

    def layers(self) -> np.ndarray:
        parts = []
        for s in self.segs:
            if isinstance(s, BatchLedger):
                parts.append(s.layer.astype(np.int8))
            else:
                parts.append(np.array([int(a.layer) for a, _ in s], dtype=np.int8))
        return np.concatenate(parts) if parts else np.zeros(0, np.int8)


def _embed(router, texts, vectors, arena):
    import torch

    if vectors is None:
        emb = router.embedder
        if hasattr(emb, "embed_device"):  # HashEmbedder: hash the batch on the GPU (bit-identical)
            return emb.embed_device(texts, arena=arena)
        if hasattr(emb, "embed_matrix"):
            V = emb.embed_matrix(texts)
        else:
            V = np.stack([np.asarray(emb.embed(t).values, dtype=np.float32) for t in texts])
        return torch.from_numpy(np.ascontiguousarray(V, dtype=np.float32)).cuda()
    return torch.as_tensor(vectors, dtype=torch.float32).cuda().contiguous()


def _is_stub(backend) -> bool:
    """The stub LLM, this package's or the reference's (same recall semantics,
    generation.py:83-115); a subclass may override recall and must be called."""
    t = type(backend)
    return t is generation.StubBackend or (t.__name__ == "StubBackend" and t.__module__ == "ragcascade.generation")


def _recall_always_rejects(backend, threshold) -> bool:
    return (_is_stub(backend) and not isinstance(backend.knowledge, generation.DeviceKnowledgeTable)
            and len(backend.knowledge) == 0 and 0.0 <= threshold <= 1.0)


def _device_recall(router):
    """The recall table whose L3 outcome is decided on the device, or None."""
    backend = router.backend
    tab = getattr(backend, "knowledge", None)
    if (_is_stub(backend) and isinstance(tab, generation.DeviceKnowledgeTable)
            and 0.0 <= router.config.recall_threshold <= 1.0):
        return tab
    return None


class _Scratch:
    """Per-router device buffers of the cascade: the seed-guard stores and the KB-row mark
    array (one int32 per knowledge-base row, restored by every pr_cascade_seeds)."""

    def __init__(self, dim: int):
        self.dim = dim
        self.stores: list[FlatIndex] = []
        self.mark = None
        self.turn = 0

    def store(self, rows_bound: int) -> FlatIndex:
        # two stores, alternating: a launched span's guard store must survive until its
        # queued scan has run, while the next span fills the other one
        if len(self.stores) < 2:
            self.stores.append(FlatIndex(dim=self.dim, capacity=rows_bound))
        s = self.stores[self.turn]
        self.turn ^= 1
        s.clear()
        return s

    def marks(self, n: int):
        import torch

        if self.mark is None or self.mark.numel() < n:
            self.mark = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
            _lib.check(_lib.load().pr_cascade_mark_init(_lib.ptr(self.mark), self.mark.numel(), _lib.stream_ptr()),
                       "mark_init")
        return self.mark


def _scratch(router, dim) -> _Scratch:
    s = getattr(router, "_cascade_scratch", None)
    if s is None or s.dim != dim:
        s = router._cascade_scratch = _Scratch(dim)
    return s


class _Span:
    """A span whose device stage has been enqueued."""

    __slots__ = ("start", "end", "size", "B", "qs", "texts", "arena", "n_pre_sc", "new_js", "prev_last",
                 "prev", "host", "event", "kb_rows_d", "kb_cnt_d", "nlist_d", "t_start", "entries", "recall",
                 "l3", "l3_val", "first", "first_of")


def _launch(router, queries, vectors, start: int, end: int, mode: int, prev: "_Span | None") -> _Span:
    """Enqueue a span's device stage (see the module doc); nothing is read back here."""
    import torch

    L = _lib.load()
    cfg = router.config
    order = cfg.probe_order()
    pos = {Lr: i for i, Lr in enumerate(order)}
    kv, sc, akm, kb = router.kv_cache, router.semantic_cache, router.adaptive_memory, router.knowledge_base
    sp = _Span()
    sp.t_start = time.perf_counter_ns()
    prof = _Prof(getattr(router, "profile_batches", False))
    sp.start, sp.end = start, end
    qs = queries[start:end]
    B = sp.size = sp.B = len(qs)
    sp.qs = qs
    texts = sp.texts = [q.text for q in qs]
    sp.entries = None
    arena = sp.arena = to_device(texts)  # one device UTF-8 arena: embedding, L1 probe, KV write-back
    Vd = _embed(router, texts, None if vectors is None else vectors[start:end], arena)
    s = _lib.stream_ptr()
    prof.mark("L.embed")
    dev = "cuda"

    # ---- window dedupe (host, texts only): an earlier write of the same text in this span
    # or in the previous one (that span is written back before this span's queries route)
    first_of = dict(zip(reversed(texts), range(B - 1, -1, -1)))  # earliest index wins (inserted last)
    first = np.fromiter(map(first_of.__getitem__, texts), dtype=np.int64, count=B)
    sp.first, sp.first_of = first, first_of
    ar = np.arange(B)
    rep = first < ar
    sp.prev_last = None
    sp.prev = prev
    if prev is not None:
        prev_last = dict(zip(prev.texts, range(prev.B)))  # latest writer in the previous span
        sp.prev_last = prev_last
        rep |= np.fromiter(map(prev_last.__contains__, texts), dtype=bool, count=B)

    prof.mark("L.dedupe")
    # ---- L2 rows write-back will create: first occurrences of texts new to the cache
    sc_index = sc.index
    sp.n_pre_sc = n_pre_sc = len(sc_index)
    with sc_index._lock:
        sc_rows = sc_index._row_by_id
        f_js = np.flatnonzero(first == ar)
        known = np.fromiter(map(sc_rows.__contains__, map(texts.__getitem__, f_js.tolist())), dtype=bool,
                            count=f_js.size)
        new_js = f_js[~known]
    sp.new_js = new_js
    prof.mark("L.new_js")
    if new_js.size:
        sc_index.extend_arrays(list(map(texts.__getitem__, new_js.tolist())), Vd[_lib.h2d(new_js)],
                               payloads=[None] * int(new_js.size), validate=False)
    sc_limit = n_pre_sc + np.searchsorted(new_js, ar, side="left")  # rows written by queries i < j
    prof.mark("L.sc_extend")

    if _ROUTE_C and not getattr(kb.index, "sharded", False):
        return _launch_c(router, sp, Vd, arena, rep, sc_limit, mode, prev, pos, prof)
    # ---- L1 probe, L2 top-1, gate + miss-list compaction: all on the device
    u8, i64 = torch.uint8, torch.int64
    kv_hit = kv_val = None
    if L1 in pos:
        kv_val, kv_hit = kv.probe_device(arena[0], arena[1], B)
    rep_d = _lib.h2d(rep.astype(np.uint8))
    l3_val = l3_d = None
    sp.recall = _device_recall(router) if L3 in pos else None
    if sp.recall is not None:
        l3_val, l3_d = sp.recall.gate_device(arena[0], arena[1], B, cfg.recall_threshold)
    r2 = None
    if L2 in pos:
        r2 = sc_index.search_batch(Vd, 1, mode=mode, validate=False, row_limit=sc_limit, count=False,
                                 floor=float(sc.threshold))
    vec_pos = min(pos.get(L4, 99), pos.get(L5, 99))
    l1_d = torch.empty(B, dtype=u8, device=dev)
    l2_d = torch.empty(B, dtype=u8, device=dev)
    lst = torch.empty(B, dtype=torch.int32, device=dev)
    nlist = torch.empty(1, dtype=torch.int32, device=dev)
    slot = torch.empty(B, dtype=torch.int32, device=dev)
    sc_cnt = r2.count if r2 is not None else None
    sc_score = r2.scores[:, 0].contiguous() if r2 is not None else None
    _lib.check(L.pr_cascade_gate(B, _lib.ptr(kv_hit), _lib.ptr(rep_d), _lib.ptr(sc_cnt), _lib.ptr(sc_score),
                                 float(sc.threshold), _lib.ptr(l3_d), int(L1 in pos and pos[L1] < vec_pos),
                                 int(L2 in pos and pos[L2] < vec_pos), int(L3 in pos and pos[L3] < vec_pos),
                                 _lib.ptr(l1_d), _lib.ptr(l2_d), _lib.ptr(lst), _lib.ptr(nlist), _lib.ptr(slot), s),
               "cascade_gate")

    prof.mark("L.l1l2l3gate")
    # ---- L5: the knowledge-base scan of the listed queries only
    sk = cfg.akm_seed_k
    kbi = kb.index
    kb_rows = torch.empty((B, sk), dtype=i64, device=dev)
    kb_raw = torch.empty((B, sk), dtype=torch.float64, device=dev)
    kb_rep = torch.empty((B, sk), dtype=torch.float64, device=dev)
    kb_cnt = torch.empty(B, dtype=torch.int32, device=dev)
    hint = int(min(B, max(1, getattr(router, "_cascade_nlist_hint", B // 2 + 1))))
    with kbi._lock:
        if getattr(kbi, "sharded", False):  # row-sharded KB: local scan + one all-gather merge (sharded.py)
            kbi.search_list(Vd, lst, nlist, B, hint, sk, mode, kb_rows, kb_raw, kb_rep, kb_cnt)
        else:
            _lib.check(L.pr_index_search_list(kbi.handle, _lib.ptr(Vd), _lib.ptr(lst), _lib.ptr(nlist), B, hint, sk,
                                              mode, None, _lib.ptr(kb_rows), _lib.ptr(kb_raw), _lib.ptr(kb_rep),
                                              _lib.ptr(kb_cnt), s), "search_list")
    sp.kb_rows_d, sp.kb_cnt_d, sp.nlist_d = kb_rows, kb_cnt, nlist
    prof.mark("L.kb")

    # ---- L4 guard: the AKM as it is now, and the superset of seeds settled before each query
    l4 = torch.zeros(B, dtype=torch.bool, device=dev)
    if L4 in pos:
        thr = akm.threshold
        if len(akm.index):
            ra = akm.index.search_batch(Vd, 1, mode=mode, validate=False, count=False, floor=float(thr))
            l4 |= (ra.count > 0) & (ra.scores[:, 0] >= thr)
        scr = _scratch(router, kbi.dim)
        prev_b = prev.B if prev is not None else 0
        out_max = (prev_b + B) * sk
        out_rows = torch.empty(out_max, dtype=i64, device=dev)
        nout = torch.empty(1, dtype=torch.int32, device=dev)
        before = torch.empty(B, dtype=i64, device=dev)
        mark = scr.marks(len(kbi))
        _lib.check(L.pr_cascade_seeds(
            _lib.ptr(prev.kb_rows_d) if prev is not None else None,
            _lib.ptr(prev.kb_cnt_d) if prev is not None else None,
            _lib.ptr(prev.nlist_d) if prev is not None else None,
            _lib.ptr(kb_rows), _lib.ptr(kb_cnt), _lib.ptr(nlist), sk, _lib.ptr(mark), _lib.ptr(out_rows), out_max,
            _lib.ptr(nout), _lib.ptr(before), s), "cascade_seeds")
        store = scr.store(out_max)
        store.append_anonymous_from(kbi, out_rows)
        lim = torch.where(slot >= 0, before[slot.clamp(min=0).long()], torch.zeros_like(before))
        rs = store.search_batch(Vd, 1, mode=mode, validate=False, row_limit=lim, count=False, floor=float(thr))
        l4 |= (rs.count > 0) & (rs.scores[:, 0] >= thr)
        l4 &= slot >= 0

    prof.mark("L.l4guard")
    # ---- the span's one read-back: outcomes + the listed queries' KB rows
    none = torch.full((B,), -1, dtype=i64, device=dev)
    cols = [l1_d.to(i64), l2_d.to(i64), slot.to(i64), l4.to(i64),
            (r2.rows[:, 0] if r2 is not None else none),
            (kv_val if kv_val is not None else none),
            kb_cnt.to(i64),
            (l3_d.to(i64) if l3_d is not None else none),
            (l3_val if l3_val is not None else none),
            nlist.to(i64)]
    packed = torch.cat([c.reshape(-1) for c in cols] + [kb_rows.reshape(-1)])
    sp.host, sp.event = pinned.ring().d2h(packed)
    prof.mark("L.pack")
    prof.merge_into(router)
    return sp


# PR_CASCADE_ROUTE=0: the span's device stage as separate calls from Python (A/B knob; a
# row-sharded knowledge base always takes that path: its scan ends in a collective)
_ROUTE_C = os.environ.get("PR_CASCADE_ROUTE", "1") != "0"


def _hv(h):
    return h.value if isinstance(h, ctypes.c_void_p) else h


def _launch_c(router, sp, Vd, arena, rep, sc_limit, mode, prev, pos, prof) -> _Span:
    """The span's device stage as ONE pr_cascade_route call (include/pentarag.h): L1 probe,
    L2 threshold top-1, gate + miss list, knowledge-base list scan, L4 guard, packed result."""
    import torch

    L = _lib.load()
    cfg = router.config
    kv, sc, akm, kb = router.kv_cache, router.semantic_cache, router.adaptive_memory, router.knowledge_base
    B, sk, kbi = sp.B, cfg.akm_seed_k, kb.index
    s = _lib.stream_ptr()
    dev, i64 = "cuda", torch.int64
    vec_pos = min(pos.get(L4, 99), pos.get(L5, 99))
    d = _lib.CascadeSpan()
    d.B, d.d_vec, d.mode = B, _lib.ptr(Vd), mode
    rep_d = _lib.h2d(rep.astype(np.uint8))
    d.d_rep = _lib.ptr(rep_d)
    if L1 in pos:
        d.kv, d.d_text, d.d_text_off = _hv(kv._h), _lib.ptr(arena[0]), _lib.ptr(arena[1])
    sp.recall = _device_recall(router) if L3 in pos else None
    l3_val = l3_d = None
    if sp.recall is not None:
        l3_val, l3_d = sp.recall.gate_device(arena[0], arena[1], B, cfg.recall_threshold)
        d.d_l3_hit, d.d_l3_val = _lib.ptr(l3_d), _lib.ptr(l3_val)
    lim_d = None
    if L2 in pos:
        lim_d = _lib.h2d(sc_limit, i64)
        d.sc, d.d_sc_limit, d.sc_threshold = _hv(sc.index.handle), _lib.ptr(lim_d), float(sc.threshold)
    d.l1_blocks = int(L1 in pos and pos[L1] < vec_pos)
    d.l2_blocks = int(L2 in pos and pos[L2] < vec_pos)
    d.l3_blocks = int(L3 in pos and pos[L3] < vec_pos)
    kb_rows = torch.empty((B, sk), dtype=i64, device=dev)
    kb_raw = torch.empty((B, sk), dtype=torch.float64, device=dev)
    kb_rep = torch.empty((B, sk), dtype=torch.float64, device=dev)
    kb_cnt = torch.empty(B, dtype=torch.int32, device=dev)
    nlist = torch.empty(1, dtype=torch.int32, device=dev)
    slot = torch.empty(B, dtype=torch.int32, device=dev)
    packed = torch.empty(9 * B + 1 + B * sk, dtype=i64, device=dev)
    d.kb, d.seed_k = _hv(kbi.handle), sk
    d.nlist_hint = int(min(B, max(1, getattr(router, "_cascade_nlist_hint", B // 2 + 1))))
    d.d_kb_rows, d.d_kb_raw, d.d_kb_rep = _lib.ptr(kb_rows), _lib.ptr(kb_raw), _lib.ptr(kb_rep)
    d.d_kb_cnt, d.d_nlist, d.d_slot, d.d_packed = _lib.ptr(kb_cnt), _lib.ptr(nlist), _lib.ptr(slot), _lib.ptr(packed)
    locks = [sc.index._lock]
    if L4 in pos:
        scr = _scratch(router, kbi.dim)
        prev_b = prev.B if prev is not None else 0
        guard = scr.store((prev_b + B) * sk)
        d.probe_l4, d.akm_rows, d.akm_threshold = 1, len(akm.index), float(akm.threshold)
        d.akm, d.guard, d.d_mark = _hv(akm.index.handle), _hv(guard.handle), _lib.ptr(scr.marks(len(kbi)))
        if prev is not None:
            d.d_prev_rows, d.d_prev_cnt, d.d_prev_n = (_lib.ptr(prev.kb_rows_d), _lib.ptr(prev.kb_cnt_d),
                                                       _lib.ptr(prev.nlist_d))
            d.prev_B = prev.B
        locks.append(akm.index._lock)
        prev_for_scratch = prev_b
    else:
        prev_for_scratch = 0
    locks.append(kbi._lock)  # last: the knowledge base may be shared by concurrent routers
    need = int(L.pr_cascade_route_scratch(B, sk, prev_for_scratch))
    buf = getattr(router, "_cascade_route_buf", None)
    if buf is None or buf.numel() < need:
        buf = router._cascade_route_buf = torch.empty(need + need // 4, dtype=torch.uint8, device=dev)
    for lk in locks:
        lk.acquire()
    try:
        _lib.check(L.pr_cascade_route(ctypes.byref(d), _lib.ptr(buf), buf.numel(), s), "cascade_route")
    finally:
        for lk in reversed(locks):
            lk.release()
    sp.kb_rows_d, sp.kb_cnt_d, sp.nlist_d = kb_rows, kb_cnt, nlist
    prof.mark("L.route")
    sp.host, sp.event = pinned.ring().d2h(packed)
    prof.mark("L.pack")
    prof.merge_into(router)
    return sp


def _discard(router, sp: _Span) -> None:
    """Drop a speculative span: its appended cache rows go (they are the newest rows)."""
    sc_index = router.semantic_cache.index
    if len(sc_index) > sp.n_pre_sc:
        sc_index.truncate(sp.n_pre_sc)


def _unpack(sp: _Span, sk: int):
    sp.event.synchronize()
    h = sp.host.copy()  # out of the pinned ring: the ledger keeps views of it
    B = sp.B
    l1, l2, slot, l4, sc_row, kv_val, kb_cnt, l3, l3_val = (h[i * B:(i + 1) * B] for i in range(9))
    nl = int(h[9 * B])
    kb_rows = h[9 * B + 1:].reshape(B, sk)
    sp.l3, sp.l3_val = l3 > 0, l3_val
    return l1.astype(bool), l2.astype(bool), slot, l4.astype(bool), sc_row, kv_val, kb_rows[:nl], kb_cnt[:nl], nl


def _finish(router, sp: _Span, *, more_follow: bool):
    """The span's host stage: decisions, answers, write-back, counters.  Returns
    (queries routed, ledger); stops before a query whose L4 outcome is uncertain."""
    cfg = router.config
    order = cfg.probe_order()
    pos = {L: i for i, L in enumerate(order)}
    backend = router.backend
    qs, texts = sp.qs, sp.texts
    sc_index = router.semantic_cache.index
    kv = router.kv_cache
    prof = _Prof(getattr(router, "profile_batches", False))
    # host work that needs no device result: the ledger shell and the span's cache entries
    ledger = BatchLedger.__new__(BatchLedger)
    now = time.monotonic_ns()
    entries = sp.entries = entries_of(texts, ledger, now)
    prof.mark("prep")
    l1, l2, slot, l4_unsure, sc_row, kv_val, kb_rows, kb_cnt, nlist = _unpack(sp, cfg.akm_seed_k)
    router._cascade_nlist_hint = max(1, nlist)
    prof.mark("wait")
    counters = {a: getattr(backend, a) for a in _BACKEND_COUNTERS if isinstance(getattr(backend, a, None), int)}
    try:
        p, serving, lat, text, conf_l, recalled = _decide(router, sp, l1, l2, slot, l4_unsure, kb_rows, kb_cnt,
                                                           prof)
    except Exception as exc:
        # the rows appended up front carry no payload yet: never leave them searchable
        # (a later L2 hit on one would serve None).  Backend counters go back to
        # where they were so the sequential re-route counts each call once.
        if len(sc_index) > sp.n_pre_sc:
            sc_index.truncate(sp.n_pre_sc)
        for a, v in counters.items():
            setattr(backend, a, v)
        raise _BackendFailed() from exc
    for j, a in recalled.items():  # before the cache hits: a later hit may copy a recalled answer
        text[j], conf_l[j] = a
    # ---- cache hits, in order: a hit serves a copy of the latest answer written for its key
    v1, v2, v5 = int(L1), int(L2), int(L5)
    sv = serving
    hit_js = np.flatnonzero((sv == v1) | (sv == v2))
    if hit_js.size:
        _serve_hits(router, sp, hit_js, sv == v1, sc_row, kv_val, text, conf_l)
    prof.mark("hits")
    conf = np.asarray(conf_l, dtype=np.float64)
    ctx_rows = CtxRows(kb_rows, slot[:p], kb_cnt, cfg.retrieval_k, sv == v5)
    probe_prefix = {}
    for L in order:
        probe_prefix[L] = tuple(_PROBE[M, "rejected" if M is L3 else "miss"] for M in order[: pos[L]])
    ledger.__init__(qs[:p], serving, lat, text, conf, ctx_rows, router.knowledge_base.index, probe_prefix)
    prof.mark("ledger")
    _writeback(router, sp, p, entries, ledger, serving, slot, kb_rows, kb_cnt, more_follow, prof)
    sp.prev = sp.prev_last = None  # the previous span is no longer read: no chain of spans stays alive
    return p, ledger


def _serve_hits(router, sp, hit_js, is_l1, sc_row, kv_val, text, conf_l):
    """Answers of the span's L1 / L2 hits, in order: a hit serves a copy of the latest
    answer written for its key (router.py:333-337 writes every routed query back) — by
    an earlier query of this span, else by the previous span, else the stored entry.

    The in-span writer of hit j is the last i < j whose text is the key: with each text
    numbered by its first occurrence in the span (``sp.first``), that is one
    searchsorted over the sorted (text number, position) pairs instead of a dict
    replayed query by query.  The per-hit gathers below run as ``map`` passes (the
    loop in C; ~2,000 hits per 4096-query span)."""
    texts = sp.texts
    B = len(texts)
    n = hit_js.size
    h1 = is_l1[hit_js]
    keys = [None] * n  # the serving layer's key of each hit
    kid = np.full(n, -1, dtype=np.int64)
    t1 = np.flatnonzero(h1)
    if t1.size:
        kid[t1] = sp.first[hit_js[t1]]
        _put(keys, t1.tolist(), map(texts.__getitem__, hit_js[t1].tolist()))
    t2 = np.flatnonzero(~h1)
    if t2.size:
        k2 = list(map(router.semantic_cache.index._ids.__getitem__, sc_row[hit_js[t2]].tolist()))
        kid[t2] = np.fromiter(map(sp.first_of.get, k2, repeat(-1)), dtype=np.int64, count=t2.size)
        _put(keys, t2.tolist(), k2)
    w = B + 1
    pairs = np.sort(sp.first * w + np.arange(B))
    at = np.searchsorted(pairs, kid * w + hit_js, side="left") - 1
    cand = pairs[np.maximum(at, 0)]
    src = np.where((kid >= 0) & (at >= 0) & (cand // w == kid), cand % w, -1)
    # written before this span: by the previous span (its entries), else the stored entry
    ext = np.flatnonzero(src < 0)
    m = ext.size
    if m:
        ej = hit_js[ext]
        keys_e = list(map(keys.__getitem__, ext.tolist()))
        ents = [None] * m
        pidx = np.full(m, -1, dtype=np.int64)
        if sp.prev_last is not None:
            pidx = np.fromiter(map(sp.prev_last.get, keys_e, repeat(-1)), dtype=np.int64, count=m)
            inprev = np.flatnonzero(pidx >= 0)
            _put(ents, inprev.tolist(), map(sp.prev.entries.__getitem__, pidx[inprev].tolist()))
        stored = pidx < 0
        s1 = np.flatnonzero(stored & h1[ext])
        _put(ents, s1.tolist(), map(router.kv_cache.entry_at, kv_val[ej[s1]].tolist()))
        s2 = np.flatnonzero(stored & ~h1[ext])
        _put(ents, s2.tolist(), map(router.semantic_cache.index.payload_at, sc_row[ej[s2]].tolist()))
        ejl = ej.tolist()
        if set(map(type, ents)) == {LedgerEntry}:
            # (ledger.text[j], ledger.conf[j]) of every entry, without a Python call each
            lgs, js = list(map(_ENT_LEDGER, ents)), list(map(_ENT_J, ents))
            _put(text, ejl, map(getitem, map(_TEXT, lgs), js))
            _put(conf_l, ejl, map(float, map(getitem, map(_CONF, lgs), js)))
        else:
            for j, e in zip(ejl, ents):
                text[j], conf_l[j] = entry_text_conf(e)
    # written earlier in this span: copies in order (a writer may itself be a hit; map
    # reads text[i] only after every earlier assignment ran)
    ins = np.flatnonzero(src >= 0)
    if ins.size:
        jl, il = hit_js[ins].tolist(), src[ins].tolist()
        _put(text, jl, map(text.__getitem__, il))
        _put(conf_l, jl, map(conf_l.__getitem__, il))


_ENT_LEDGER, _ENT_J = itemgetter(1), itemgetter(2)
_TEXT, _CONF, _ANSWER = attrgetter("text"), attrgetter("conf"), attrgetter("answer")


def _put(lst: list, idx, vals) -> None:
    """lst[i] = v for the pairs in order (consumed lazily: one pass in C)."""
    deque(map(lst.__setitem__, idx, vals), maxlen=0)


def _decide(router, sp, l1, l2, slot, l4_unsure, kb_rows, kb_cnt, prof):
    """Decision pass, vectorised over the span; answers of retrieval and recall."""
    cfg = router.config
    order = cfg.probe_order()
    pos = {L: i for i, L in enumerate(order)}
    backend = router.backend
    kb = router.knowledge_base
    qs, B = sp.qs, sp.B
    # a span stops before the first query whose L4 outcome is not certain (decided from
    # L1/L2 alone, so no backend side effect happens for it in batch mode)
    stop = B
    if L4 in pos:
        reach4 = l4_unsure.copy()
        for L in order[: pos[L4]]:
            if L is L1:
                reach4 &= ~l1
            elif L is L2:
                reach4 &= ~l2
        hits = np.flatnonzero(reach4)
        if hits.size:
            stop = int(hits[0])
    p = stop
    serving = np.zeros(p, dtype=np.int8)
    reach = np.ones(p, dtype=bool)
    recalled = {}
    for L in order:
        if L is L1:
            h = reach & l1[:p]
        elif L is L2:
            h = reach & l2[:p]
        elif L is L3 and sp.recall is not None:
            # decided on the device (pr_recall_gate); every query reaching L3 is one recall call
            h = reach & sp.l3[:p]
            backend.recall_calls += int(reach.sum())
            entry_at = sp.recall.entry_at
            for j, v in zip(np.flatnonzero(h).tolist(), sp.l3_val[:p][h].tolist()):
                e = entry_at(v)
                recalled[j] = (e.answer, e.confidence)
        elif L is L3 and _recall_always_rejects(backend, cfg.recall_threshold):
            # the stub LLM with an empty recall table rejects every query (generation.py);
            # only its call counter moves
            h = np.zeros(p, dtype=bool)
            backend.recall_calls += int(reach.sum())
        elif L is L3:
            h = np.zeros(p, dtype=bool)
            for j in np.flatnonzero(reach):
                rec = generation.memory_recall(backend, qs[j], cfg.recall_threshold)
                if rec is not None:
                    h[j] = True
                    recalled[int(j)] = (rec.text, rec.confidence)
        elif L is L4:
            h = np.zeros(p, dtype=bool)
        else:
            h = reach.copy()
        serving[h] = int(L)
        reach &= ~h
    prof.mark("decide")
    wall = (time.perf_counter_ns() - sp.t_start) / 1e9
    lm = router.latency_model
    if lm is None:
        lat = np.full(p, wall / max(1, p))
    elif hasattr(lm, "sample_many"):
        lat = np.asarray(lm.sample_many(serving), dtype=np.float64)
    else:
        lat = np.fromiter((lm.sample(LayerTag(int(v))) for v in serving), dtype=np.float64, count=p)
    text: list = [None] * p
    conf_l = [0.0] * p
    k_ctx = cfg.retrieval_k
    v5 = int(L5)
    # retrieval answers first: they depend on no other query of the span.  The stub LLM
    # answers with the top passage's annotation (generation.py:83-115): computed directly
    # (exact type: a subclass may override generate_with_context and must be called)
    stub = type(backend) is generation.StubBackend and 0.0 <= backend.context_confidence <= 1.0
    l5_js = np.flatnonzero(serving == v5).tolist()
    if l5_js:
        l5_slots = slot[l5_js]
        if stub:
            # top passage of each query, its answer, else its first sentence: map passes
            # (the loop in C) over the ~2,000 retrieval answers of a 4096-query span
            kbi = kb.index
            rows = kb_rows[l5_slots, 0].tolist()
            pl = getattr(kbi, "_payloads", None)
            tops = list(map(pl.__getitem__, rows)) if pl is not None else None
            if tops is None or any(map(is_, tops, repeat(_DEFERRED))):
                tops = list(map(kbi.payload_at, rows))
            ans = list(map(_ANSWER, tops))
            if not all(ans):
                first_sentence = generation.first_sentence
                ans = [a if a else first_sentence(t.text) for a, t in zip(ans, tops)]
            _put(text, l5_js, ans)
            _put(conf_l, l5_js, repeat(backend.context_confidence, len(l5_js)))
            backend.context_calls += len(l5_js)
        else:
            for j, s5 in zip(l5_js, l5_slots.tolist()):
                passages = [kb.index.payload_at(int(r)) for r in kb_rows[s5, : min(k_ctx, int(kb_cnt[s5]))]]
                a = generation.generate_with_context(backend, qs[j], passages, L5)
                text[j], conf_l[j] = a.text, a.confidence
    prof.mark("answers")
    return p, serving, lat, text, conf_l, recalled


def _writeback(router, sp, p, entries, ledger, serving, slot, kb_rows, kb_cnt, more_follow, prof):
    """Write-back (router.py:333-337) and counters of the span's first p queries."""
    cfg = router.config
    order = cfg.probe_order()
    pos = {L: i for i, L in enumerate(order)}
    kv, sc, akm, kb = router.kv_cache, router.semantic_cache, router.adaptive_memory, router.knowledge_base
    sc_index = sc.index
    texts = sp.texts
    kv.put_entries(texts[:p], entries[:p], arena=sp.arena)
    prof.mark("wb.kv")
    if p < sp.B:
        # a stopped span: the rows of its unrouted queries go, and with them every row a
        # speculative next span appended after them (that span is discarded)
        n_new_kept = int(np.searchsorted(sp.new_js, p, side="left"))
        if sp.n_pre_sc + n_new_kept < len(sc_index):
            sc_index.truncate(sp.n_pre_sc + n_new_kept)
    with sc._lock, sc_index._lock:
        payloads, rowmap = sc_index._payloads, sc_index._row_by_id
        # in order (the last write of a text wins), the loop run by map in C
        deque(map(payloads.__setitem__, map(rowmap.__getitem__, texts[:p]), entries), maxlen=0)
        prof.mark("wb.sc_payloads")
        seq = sc._seq
        sc._recency.update(zip(texts[:p], range(seq + 1, seq + p + 1)))
        sc._seq = seq + p
    prof.mark("wb.sc")
    # AKM: seeds of retrieval-served queries settle before the next query routes
    # (device-to-device from KB rows, dedupe by id, no overwrite).  The last query's
    # seeds stay pending, exactly as after route(), unless more queries of this call
    # follow — the next one would settle them first anyway.
    upto = p if (more_follow or p < sp.B) else max(p - 1, 0)
    l5_slots = slot[np.flatnonzero(serving[:upto] == int(L5))]
    if l5_slots.size:
        # row-major boolean selection = the per-query seed lists concatenated in order
        valid = np.arange(kb_rows.shape[1])[None, :] < kb_cnt[l5_slots][:, None]
        akm.settle_from_rows(kb.index, kb_rows[l5_slots][valid])
    if upto < p and serving[p - 1] == int(L5):
        s = slot[p - 1]
        akm.enqueue([kb.index.payload_at(int(r)) for r in kb_rows[s, : kb_cnt[s]]])
    prof.mark("wb.akm")
    # ---- counters: a layer is probed by every query served at or after it
    pos_of_code = np.full(max(int(L) for L in LayerTag) + 1, -1, dtype=np.int64)
    for L in order:
        pos_of_code[int(L)] = pos[L]
    served_pos = pos_of_code[serving.astype(np.int64)]
    for L in order:
        probed = int((served_pos >= pos[L]).sum())
        hit = int((serving == int(L)).sum())
        if L is L1:
            kv.hits += hit
            kv.misses += probed - hit
        elif L is L2:
            sc.hits += hit
            sc.misses += probed - hit
            sc_index.search_count += probed
        elif L is L4:
            akm.misses += probed
            akm.index.search_count += probed
        elif L is L5:
            with kb.index._lock:  # the knowledge base may be shared by concurrently replayed sessions
                kb.index.search_count += probed
    router.trace.extend_ledger(ledger)
    prof.mark("writeback")
    if prof.enabled:
        hist = getattr(router, "batch_profile", None)
        if hist is None:
            hist = router.batch_profile = {}
        for k, v in prof.times.items():
            hist[k] = hist.get(k, 0.0) + v
        router.batch_profile_log = getattr(router, "batch_profile_log", []) + [dict(prof.times)]


_BACKEND_COUNTERS = ("recall_calls", "context_calls")


class _BackendFailed(Exception):
    """Raised by _finish after rolling its store mutations back."""


class _Prof:
    """Optional stage timer (wall time of the host stage's parts)."""

    def __init__(self, enabled: bool):
        self.enabled = enabled
        self.times: dict[str, float] = {}
        self._t = time.perf_counter()

    def merge_into(self, router) -> None:
        if not self.enabled:
            return
        hist = getattr(router, "batch_profile", None)
        if hist is None:
            hist = router.batch_profile = {}
        for k, v in self.times.items():
            hist[k] = hist.get(k, 0.0) + v

    def mark(self, name: str) -> None:
        if not self.enabled:
            return
        t = time.perf_counter()
        self.times[name] = self.times.get(name, 0.0) + (t - self._t)
        self._t = t
