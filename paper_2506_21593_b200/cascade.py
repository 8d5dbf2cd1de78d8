"""Batched, sequential-equivalent routing.

``route_batch(router, queries)`` returns exactly what
``[router.route(q) for q in queries]`` returns — answers, trace events,
store contents and every counter — while doing the per-layer work as a few
batched device calls:

* L1 (fixed KV): one fused fingerprint+probe kernel over the batch's UTF-8
  arena; a query also hits if an EARLIER query in the batch had the same text,
  because every served answer is written back before the next query
  (router.py:333-337) — a causal first-occurrence dedupe.
* L2 (semantic cache): the first occurrence of every new text is appended to
  the cache store up front (that is what write-back will do), and ONE
  row-limited top-1 search (pr_index_search_ex) lets query j see exactly the
  pre-batch rows plus the rows written by queries i < j.  Ties keep the
  earlier row, as sequential upserts would.
* L4 (adaptive memory) depends on which earlier queries were served by L5
  (their seeds are settled before the next query, router.py:284-285), a
  routing OUTCOME.  The batch proves L4 misses instead: top-1 over the
  pre-batch AKM and over a superset of every seed any earlier query of the
  batch could contribute (row-limited search over a scratch store gathered
  device-to-device from knowledge-base rows).  If that bound reaches the AKM
  threshold for some query, the batch stops before it and that query is
  routed by ``router.route`` exactly; batching resumes after it.
* L5: one top-seed_k search for every query that can reach it.

All scores are the exact fp64 reference scores (bit-identical), so every
threshold decision is the reference's.  The decision pass over the batch is
O(B) host work; latencies come from the router's synthetic latency model in
query order (or the batch wall time split evenly when there is none).

Regimes that need per-query state changes inside the batch fall back to
``route`` per query: no knowledge base / NAIVE_RAG disabled (queries may
miss every layer and skip write-back), capped caches (LRU eviction), or a
non-deterministic AKM settle thread.
"""
from __future__ import annotations

import time

import numpy as np

from . import generation
from .caches import CacheEntry, FixedKVCache, SemanticCache
from .index import MODE_AUTO, FlatIndex, first_occurrences
from .knowledge import AdaptiveKnowledgeMemory
from .records import AnswerRecord, LayerTag
from .errors import CascadeError
from .ledger import BatchLedger, CtxRows, LedgerEntry, entry_text_conf
from .router import LayerProbe
from .textarena import to_device

L1, L2, L3, L4, L5 = (LayerTag.FIXED_KV, LayerTag.SEMANTIC_CACHE, LayerTag.MEMORY_RECALL,
                      LayerTag.ADAPTIVE_MEMORY, LayerTag.NAIVE_RAG)
# immutable probe records shared by every routed query (only the serving
# layer's probe carries a latency and is built per query)
_PROBE = {(L, o): LayerProbe(L, o) for L in LayerTag for o in ("hit", "miss", "rejected")}


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
                capture_errors: bool = False):
    """Route ``queries`` in order; see the module docstring.  Returns the list
    of (AnswerRecord, RouteTraceEvent), or with ``materialize=False`` a
    ``RoutedBatch`` of columnar segments (objects built only on access).

    ``capture_errors``: a query whose ``route`` raises a CascadeError (e.g.
    AllLayersMissed, router.py:309-323 — no write-back happens for it) gets the
    exception object as its result and the batch continues, exactly like
    independent ``route`` calls would (service micro-batching)."""
    segs = []
    i, n = 0, len(queries)
    stats = {"batched": 0, "sequential": 0, "splits": 0}

    def one(q):
        if not capture_errors:
            return router.route(q)
        try:
            return router.route(q)
        except CascadeError as exc:
            return exc

    while i < n:
        if not batchable(router):
            segs.append([one(queries[i])])
            stats["sequential"] += 1
            i += 1
            continue
        V = None if vectors is None else vectors[i:]
        remaining = n - i
        try:
            done, ledger = _route_prefix(router, queries[i:], V, mode)
        except _BackendFailed:
            # a backend call raised mid-batch: every store mutation of the batch was rolled
            # back, so route the span one query at a time — the failing query raises (or is
            # captured) exactly where independent route() calls would raise
            for q in queries[i:]:
                segs.append([one(q)])
            stats["sequential"] += remaining
            break
        if done:
            segs.append(ledger)
        stats["batched"] += done
        i += done
        if done < remaining:
            # the next query's AKM outcome is not certain in batch: route it exactly
            segs.append([one(queries[i])])
            stats["sequential"] += 1
            stats["splits"] += 1
            i += 1
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


def _recall_always_rejects(backend, threshold) -> bool:
    return (type(backend) is generation.StubBackend and len(backend.knowledge) == 0
            and 0.0 <= threshold <= 1.0)


def _row_scratch(router, n: int) -> np.ndarray:
    buf = getattr(router, "_row_pos", None)
    if buf is None or buf.size < n:
        buf = router._row_pos = np.empty(max(n, 1), dtype=np.int32)
    return buf


def _seed_scratch(router, dim, rows_bound: int) -> FlatIndex:
    """The router's reusable seed store, reserved for the batch's worst case up
    front (growing it mid-run would reallocate between two dependent searches)."""
    s = getattr(router, "_seed_scratch", None)
    if s is None or s.dim != dim:
        s = FlatIndex(dim=dim, capacity=rows_bound)
        router._seed_scratch = s
    s.clear()
    return s


def _route_prefix(router, qs, vectors, mode):
    import torch

    cfg = router.config
    order = cfg.probe_order()
    pos = {L: i for i, L in enumerate(order)}
    kv, sc, akm, kb = router.kv_cache, router.semantic_cache, router.adaptive_memory, router.knowledge_base
    backend = router.backend
    t_start = time.perf_counter_ns()
    prof = _Prof(getattr(router, "profile_batches", False))
    akm.settle()  # the first route() of the run would settle the pre-batch queue (router.py:284-285)

    B = len(qs)
    texts = [q.text for q in qs]
    arena = to_device(texts)  # one device UTF-8 arena: embedding, L1 probe, KV write-back
    Vd = _embed(router, texts, vectors, arena)
    ar = np.arange(B)

    prof.mark("settle+embed")
    # ---- L1: pre-batch probe + causal first-occurrence dedupe
    first_of = {t: j for j, t in zip(range(B - 1, -1, -1), reversed(texts))}  # earliest index wins
    first = np.fromiter(map(first_of.__getitem__, texts), dtype=np.int64, count=B)
    l1 = np.zeros(B, dtype=bool)
    kv_val = np.full(B, -1, dtype=np.int64)
    if L1 in pos:
        vals, hit = kv.probe_device(arena[0], arena[1], B)
        kv_val = vals.cpu().numpy()
        l1 = hit.cpu().numpy().astype(bool) | (first < ar)

    prof.mark("l1")
    # ---- L2: append the rows write-back will create, then one row-limited top-1 search
    sc_index = sc.index
    n_pre_sc = len(sc_index)
    with sc_index._lock:
        sc_rows = sc_index._row_by_id
        new_js = np.array([j for j in np.flatnonzero(first == ar).tolist() if texts[j] not in sc_rows],
                          dtype=np.int64)
    if new_js.size:
        sc_index.extend_arrays([texts[j] for j in new_js], Vd[torch.from_numpy(new_js).cuda()],
                               payloads=[None] * int(new_js.size), validate=False)
    counters = {a: getattr(backend, a) for a in _BACKEND_COUNTERS if isinstance(getattr(backend, a, None), int)}
    try:
        return _route_rest(router, qs, texts, arena, Vd, mode, prof, t_start, first, l1, kv_val, sc_index,
                           n_pre_sc, new_js)
    except _WritebackFailed as exc:
        raise exc.__cause__
    except Exception as exc:
        # the rows appended above carry no payload yet: never leave them searchable
        # (a later L2 hit on one would serve None).  Backend counters go back to
        # where they were so the sequential re-route counts each call once.
        if len(sc_index) > n_pre_sc:
            sc_index.truncate(n_pre_sc)
        for a, v in counters.items():
            setattr(backend, a, v)
        raise _BackendFailed() from exc


def _route_rest(router, qs, texts, arena, Vd, mode, prof, t_start, first, l1, kv_val, sc_index, n_pre_sc, new_js):
    import torch

    cfg = router.config
    order = cfg.probe_order()
    pos = {L: i for i, L in enumerate(order)}
    kv, sc, akm, kb = router.kv_cache, router.semantic_cache, router.adaptive_memory, router.knowledge_base
    backend = router.backend
    B = len(qs)
    ar = np.arange(B)
    sc_limit = n_pre_sc + np.searchsorted(new_js, ar, side="left")  # rows written by queries i < j
    l2 = np.zeros(B, dtype=bool)
    sc_row = np.full(B, -1, dtype=np.int64)
    # only queries that actually probe L2 are searched (an L1 hit in front of it ends the cascade)
    need2 = ~l1 if (L1 in pos and L2 in pos and pos[L1] < pos[L2]) else np.ones(B, dtype=bool)
    js2 = np.nonzero(need2)[0]
    if L2 in pos and js2.size:
        sel = torch.from_numpy(js2).cuda()
        r = sc_index.search_batch(Vd[sel], 1, mode=mode, validate=False, row_limit=sc_limit[js2], count=False)
        prof.note("sc", sc_index)
        sc_row[js2] = r.rows[:, 0].cpu().numpy()
        l2[js2] = (r.count.cpu().numpy() > 0) & (r.scores[:, 0].cpu().numpy() >= sc.threshold)

    prof.mark("l2")

    def host_prep():
        """Host work that needs no knowledge-base result (runs while the KB scan is in
        flight): the batch's ledger shell, its cache entries, and for every L1/L2 hit
        candidate the latest earlier query of the batch that wrote the same key."""
        ledger = BatchLedger.__new__(BatchLedger)
        now = time.monotonic_ns()
        entries = [LedgerEntry(t, ledger, j, now) for j, t in enumerate(texts)]
        l1l, l2l, scr = l1.tolist(), l2.tolist(), sc_row.tolist()
        l1_first = L1 in pos and (L2 not in pos or pos[L1] < pos[L2])
        sc_ids = sc_index._ids
        src = [-1] * B
        latest: dict[str, int] = {}
        for j, t in enumerate(texts):
            a, b = l1l[j], l2l[j]
            if a or b:  # the serving one of L1 / L2 is the earlier of the two in probe order
                src[j] = latest.get(t if (a and (l1_first or not b)) else sc_ids[scr[j]], -1)
            latest[t] = j
        return ledger, entries, src

    prep = None
    # ---- L4/L5 speculation for every query that can reach them
    vec_pos = min(pos.get(L4, 99), pos.get(L5, 99))
    blocked = np.zeros(B, dtype=bool)
    if L1 in pos and pos[L1] < vec_pos:
        blocked |= l1
    if L2 in pos and pos[L2] < vec_pos:
        blocked |= l2
    spec = np.nonzero(~blocked)[0]
    slot = np.full(B, -1, dtype=np.int64)
    slot[spec] = np.arange(spec.size)
    kb_rows = np.zeros((0, cfg.akm_seed_k), dtype=np.int64)
    kb_cnt = np.zeros(0, dtype=np.int32)
    l4_unsure = np.zeros(B, dtype=bool)
    if spec.size:
        Vs = Vd[torch.from_numpy(spec).cuda()]
        r = kb.index.search_batch(Vs, cfg.akm_seed_k, mode=mode, validate=False, count=False)
        prof.note("kb", kb.index)
        # the pre-batch AKM probe does not depend on the KB results: queue it behind the scan
        ra = None
        if L4 in pos and len(akm.index):
            ra = akm.index.search_batch(Vs, 1, mode=mode, validate=False, count=False)
            prof.note("akm", akm.index)
        prep = host_prep()
        kb_rows, kb_cnt = r.rows.cpu().numpy(), r.count.cpu().numpy()
        if L4 in pos:
            thr = akm.threshold
            if ra is not None:
                l4_unsure[spec] |= (ra.count.cpu().numpy() > 0) & (ra.scores[:, 0].cpu().numpy() >= thr)
            # superset of in-batch seeds: every seed of every earlier speculative query
            # row-major boolean selection = the per-query seed lists concatenated in order
            seed_rows = kb_rows[np.arange(kb_rows.shape[1])[None, :] < kb_cnt[:, None]]
            seeds_before = np.concatenate([[0], np.cumsum(kb_cnt)[:-1]]).astype(np.int64)
            if seed_rows.size:
                # keep the first occurrence of each KB row: query j sees the same SET of
                # vectors (a repeat only becomes visible after its first copy), and the
                # scratch loses its bit-identical duplicates, which tie at every score
                first_pos = first_occurrences(seed_rows, _row_scratch(router, len(kb.index)))
                seeds_before = np.searchsorted(first_pos, seeds_before, side="left").astype(np.int64)
                seed_rows = seed_rows[first_pos]
                scratch = _seed_scratch(router, kb.index.dim, B * cfg.akm_seed_k)
                scratch.append_anonymous_from(kb.index, seed_rows)
                rs = scratch.search_batch(Vs, 1, mode=mode, validate=False, row_limit=seeds_before, count=False)
                prof.note("seeds", scratch)
                l4_unsure[spec] |= (rs.count.cpu().numpy() > 0) & (rs.scores[:, 0].cpu().numpy() >= thr)

    prof.mark("l4+l5")
    # ---- decision pass, vectorised over the batch.  A batch stops before the
    # first query whose L4 outcome is not certain (decided from L1/L2 alone, so
    # no backend side effect happens for it in batch mode)
    stop = B
    if L4 in pos:
        reach4 = l4_unsure.copy()
        for L in order[: pos[L4]]:
            if L is L1:
                reach4 &= ~l1
            elif L is L2:
                reach4 &= ~l2
        hits = np.nonzero(reach4)[0]
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
        elif L is L3 and _recall_always_rejects(backend, cfg.recall_threshold):
            # the stub LLM with an empty recall table rejects every query (generation.py);
            # only its call counter moves
            h = np.zeros(p, dtype=bool)
            backend.recall_calls += int(reach.sum())
        elif L is L3:
            h = np.zeros(p, dtype=bool)
            for j in np.nonzero(reach)[0]:
                rec = generation.memory_recall(backend, qs[j], cfg.recall_threshold)
                if rec is not None:
                    h[j] = True
                    recalled[int(j)] = rec
        elif L is L4:
            h = np.zeros(p, dtype=bool)
        else:
            h = reach.copy()
        serving[h] = int(L)
        reach &= ~h

    prof.mark("decide")
    # ---- answers as columns; objects are materialised lazily (ledger.py)
    wall = (time.perf_counter_ns() - t_start) / 1e9
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
    v1, v2, v5 = int(L1), int(L2), int(L5)
    sv = serving[:p]
    # L5 answers first: they depend on no other query of the batch.  The stub LLM
    # answers with the top passage's annotation (generation.py:83-115): compute that
    # directly instead of building a context answer object per query
    # exact type: a subclass may override generate_with_context (and must be called)
    stub = type(backend) is generation.StubBackend and 0.0 <= backend.context_confidence <= 1.0
    l5_js = np.flatnonzero(sv == v5).tolist()
    if l5_js:
        l5_slots = slot[l5_js]
        if stub:
            payload_at, first_sentence = kb.index.payload_at, generation.first_sentence
            cc = backend.context_confidence
            for j, r in zip(l5_js, kb_rows[l5_slots, 0].tolist()):
                top = payload_at(r)
                text[j] = top.answer if top.answer else first_sentence(top.text)
                conf_l[j] = cc
            backend.context_calls += len(l5_js)
        else:
            for j, s5 in zip(l5_js, l5_slots.tolist()):
                passages = [kb.index.payload_at(int(r)) for r in kb_rows[s5, : min(k_ctx, int(kb_cnt[s5]))]]
                a = generation.generate_with_context(backend, qs[j], passages, L5)
                text[j], conf_l[j] = a.text, a.confidence
    for j, a in recalled.items():
        text[j], conf_l[j] = a.text, a.confidence
    # cache hits, in order: a hit serves a copy of the latest answer written for its key
    if prep is None:
        prep = host_prep()
    ledger, entries, src = prep
    hit_js = np.flatnonzero((sv == v1) | (sv == v2)).tolist()
    if hit_js:
        codes, scr, kvv = sv.tolist(), sc_row[:p].tolist(), kv_val[:p].tolist()
        kv_entry, sc_payload = kv.entry_at, sc_index.payload_at
        for j in hit_js:  # ascending: an earlier writer's answer is already filled
            i = src[j]
            if i >= 0:
                text[j], conf_l[j] = text[i], conf_l[i]
            elif codes[j] == v1:
                text[j], conf_l[j] = entry_text_conf(kv_entry(kvv[j]))
            else:
                text[j], conf_l[j] = entry_text_conf(sc_payload(scr[j]))
    conf = np.asarray(conf_l, dtype=np.float64)
    ctx_rows = CtxRows(kb_rows, slot[:p], kb_cnt, k_ctx, sv == v5)
    probe_prefix = {}
    for L in order:
        pre = []
        for M in order[: pos[L]]:
            pre.append(_PROBE[M, "rejected" if M is L3 else "miss"])
        probe_prefix[L] = tuple(pre)
    ledger.__init__(qs[:p], serving, lat, text, conf, ctx_rows, kb.index, probe_prefix)

    prof.mark("materialise")
    # ---- write-back (router.py:333-337): KV in order (last write wins), SC payloads.
    # Every backend call of the batch happened above; a failure from here on is not a
    # per-query error and is not retried query by query.
    try:
        return _writeback(router, qs, texts, arena, prof, p, entries, ledger, serving, slot, kb_rows, kb_cnt,
                          sc_index, n_pre_sc, new_js)
    except Exception as exc:
        raise _WritebackFailed() from exc


def _writeback(router, qs, texts, arena, prof, p, entries, ledger, serving, slot, kb_rows, kb_cnt, sc_index,
               n_pre_sc, new_js):
    cfg = router.config
    order = cfg.probe_order()
    pos = {L: i for i, L in enumerate(order)}
    kv, sc, akm, kb = router.kv_cache, router.semantic_cache, router.adaptive_memory, router.knowledge_base
    del entries[p:]
    kv.put_entries(texts[:p], entries, arena=arena)
    prof.mark("wb.kv")
    n_new_kept = int(np.searchsorted(new_js, p, side="left"))
    if n_pre_sc + n_new_kept < len(sc_index):
        sc_index.truncate(n_pre_sc + n_new_kept)
    with sc._lock, sc_index._lock:
        payloads, rowmap = sc_index._payloads, sc_index._row_by_id
        for t, e in zip(texts[:p], entries):
            payloads[rowmap[t]] = e  # in order: the last write of a text wins
        seq = sc._seq
        sc._recency.update(zip(texts[:p], range(seq + 1, seq + p + 1)))
        sc._seq = seq + p
    prof.mark("wb.sc")
    # AKM: seeds of L5 queries before the last were settled by the following
    # route() calls (device-to-device from KB rows, dedupe by id, no overwrite);
    # the final query's seeds are still pending, exactly as after route()
    l5_slots = slot[np.flatnonzero(serving[: max(p - 1, 0)] == int(L5))]
    if l5_slots.size:
        # row-major boolean selection = the per-query seed lists concatenated in order
        valid = np.arange(kb_rows.shape[1])[None, :] < kb_cnt[l5_slots][:, None]
        akm.settle_from_rows(kb.index, kb_rows[l5_slots][valid])
    if p and serving[p - 1] == int(L5):
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
    return p, ledger


_BACKEND_COUNTERS = ("recall_calls", "context_calls")


class _BackendFailed(Exception):
    """Raised by _route_prefix after rolling its store mutations back."""


class _WritebackFailed(Exception):
    """Wraps a write-back failure so it passes the rollback handler unchanged."""


class _Prof:
    """Optional stage timer (synchronises the device at each mark)."""

    def __init__(self, enabled: bool):
        self.enabled = enabled
        self.times: dict[str, float] = {}
        self._t = time.perf_counter()

    def note(self, name: str, index) -> None:
        if not self.enabled:
            return
        st = index.stats()
        self.mark(name)
        self.times[f"{name}.rows"] = self.times.get(f"{name}.rows", 0) + len(index)
        self.times[f"{name}.queries"] = self.times.get(f"{name}.queries", 0) + st.queries
        self.times[f"{name}.fallback"] = self.times.get(f"{name}.fallback", 0) + st.fallback
        self.times[f"{name}.collected"] = self.times.get(f"{name}.collected", 0) + st.collected
        self.times[f"{name}.tensor_path"] = self.times.get(f"{name}.tensor_path", 0) + (st.path == 2)
        self.times[f"{name}.i8_path"] = self.times.get(f"{name}.i8_path", 0) + (st.path == 3)
        self.times[f"{name}.appended"] = self.times.get(f"{name}.appended", 0) + st.appended
        self.times[f"{name}.rescored"] = self.times.get(f"{name}.rescored", 0) + st.candidates

    def mark(self, name: str) -> None:
        if not self.enabled:
            return
        import torch

        torch.cuda.synchronize()
        t = time.perf_counter()
        self.times[name] = self.times.get(name, 0.0) + (t - self._t)
        self._t = t
