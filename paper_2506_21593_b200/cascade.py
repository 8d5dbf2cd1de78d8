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
from .caches import CacheEntry, FixedKVCache, SemanticCache, encode_texts
from .index import MODE_AUTO, FlatIndex
from .knowledge import AdaptiveKnowledgeMemory
from .records import AnswerRecord, LayerTag
from .router import LayerProbe, RouteTraceEvent

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


def route_batch(router, queries, vectors=None, *, mode: int = MODE_AUTO):
    """Route ``queries`` in order; see the module docstring."""
    out = []
    i, n = 0, len(queries)
    stats = {"batched": 0, "sequential": 0, "splits": 0}
    while i < n:
        if not batchable(router):
            out.append(router.route(queries[i]))
            stats["sequential"] += 1
            i += 1
            continue
        V = None if vectors is None else vectors[i:]
        remaining = n - i
        done, res = _route_prefix(router, queries[i:], V, mode)
        out.extend(res)
        stats["batched"] += done
        i += done
        if done < remaining:
            # the next query's AKM outcome is not certain in batch: route it exactly
            out.append(router.route(queries[i]))
            stats["sequential"] += 1
            stats["splits"] += 1
            i += 1
    router.last_batch_stats = stats
    return out


def _embed(router, texts, vectors):
    import torch

    if vectors is None:
        emb = router.embedder
        if hasattr(emb, "embed_matrix"):
            V = emb.embed_matrix(texts)
        else:
            V = np.stack([np.asarray(emb.embed(t).values, dtype=np.float32) for t in texts])
        return torch.from_numpy(np.ascontiguousarray(V, dtype=np.float32)).cuda()
    return torch.as_tensor(vectors, dtype=torch.float32).cuda().contiguous()


def _seed_scratch(router, dim) -> FlatIndex:
    s = getattr(router, "_seed_scratch", None)
    if s is None or s.dim != dim:
        s = FlatIndex(dim=dim)
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
    Vd = _embed(router, texts, vectors)
    ar = np.arange(B)

    prof.mark("settle+embed")
    # ---- L1: pre-batch probe + causal first-occurrence dedupe
    first_of: dict[str, int] = {}
    first = np.fromiter((first_of.setdefault(t, j) for j, t in enumerate(texts)), dtype=np.int64, count=B)
    l1 = np.zeros(B, dtype=bool)
    kv_val = np.full(B, -1, dtype=np.int64)
    if L1 in pos:
        data, off = encode_texts(texts)
        vals, hit = kv.probe_device(torch.from_numpy(data).cuda(), torch.from_numpy(off).cuda(), B)
        kv_val = vals.cpu().numpy()
        l1 = hit.cpu().numpy().astype(bool) | (first < ar)

    prof.mark("l1")
    # ---- L2: append the rows write-back will create, then one row-limited top-1 search
    sc_index = sc.index
    n_pre_sc = len(sc_index)
    new_js = np.array([j for j in range(B) if first[j] == j and texts[j] not in sc_index], dtype=np.int64)
    if new_js.size:
        sc_index.extend_arrays([texts[j] for j in new_js], Vd[torch.from_numpy(new_js).cuda()],
                               payloads=[None] * int(new_js.size), validate=False)
    sc_limit = n_pre_sc + np.searchsorted(new_js, ar, side="left")  # rows written by queries i < j
    l2 = np.zeros(B, dtype=bool)
    sc_row = np.full(B, -1, dtype=np.int64)
    if L2 in pos and B:
        r = sc_index.search_batch(Vd, 1, mode=mode, validate=False, row_limit=sc_limit, count=False)
        prof.note("sc", sc_index)
        sc_row = r.rows[:, 0].cpu().numpy()
        l2 = (r.count.cpu().numpy() > 0) & (r.scores[:, 0].cpu().numpy() >= sc.threshold)

    prof.mark("l2")
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
        kb_rows, kb_cnt = r.rows.cpu().numpy(), r.count.cpu().numpy()
        if L4 in pos:
            thr = akm.threshold
            if len(akm.index):
                ra = akm.index.search_batch(Vs, 1, mode=mode, validate=False, count=False)
                prof.note("akm", akm.index)
                l4_unsure[spec] |= (ra.count.cpu().numpy() > 0) & (ra.scores[:, 0].cpu().numpy() >= thr)
            # superset of in-batch seeds: every seed of every earlier speculative query
            seed_rows = np.concatenate([kb_rows[s, : kb_cnt[s]] for s in range(spec.size)]) \
                if spec.size else np.zeros(0, np.int64)
            seeds_before = np.concatenate([[0], np.cumsum(kb_cnt)[:-1]]).astype(np.int64)
            if seed_rows.size:
                scratch = _seed_scratch(router, kb.index.dim)
                scratch.append_rows_from(kb.index, seed_rows, [str(i) for i in range(seed_rows.size)],
                                         [None] * seed_rows.size)
                rs = scratch.search_batch(Vs, 1, mode=mode, validate=False, row_limit=seeds_before, count=False)
                prof.note("seeds", scratch)
                l4_unsure[spec] |= (rs.count.cpu().numpy() > 0) & (rs.scores[:, 0].cpu().numpy() >= thr)

    prof.mark("l4+l5")
    # ---- decision pass (query order), stopping before an uncertain L4 probe
    p = B
    serving, probes_all = [], []
    recalled = {}
    for j in range(B):
        if L4 in pos and l4_unsure[j]:
            reaches = all(not ((L is L1 and l1[j]) or (L is L2 and l2[j])) for L in order[: pos[L4]])
            if reaches:
                p = j
                break
        probes, hit_layer = [], None
        for L in order:
            if L is L1:
                ok = bool(l1[j])
            elif L is L2:
                ok = bool(l2[j])
            elif L is L3:
                rec = generation.memory_recall(backend, qs[j], cfg.recall_threshold)
                ok = rec is not None
                if ok:
                    recalled[j] = rec
                probes.append(_PROBE[L, "hit" if ok else "rejected"])
                if ok:
                    hit_layer = L
                    break
                continue
            elif L is L4:
                ok = False
            else:
                ok = True
            probes.append(_PROBE[L, "hit" if ok else "miss"])
            if ok:
                hit_layer = L
                break
        serving.append(hit_layer)
        probes_all.append(probes)

    prof.mark("decide")
    # ---- materialise answers, write back, account (exactly as p sequential routes)
    wall = (time.perf_counter_ns() - t_start) / 1e9
    synthetic = router.latency_model is not None
    latest: dict[str, object] = {}
    answers, events = [], []
    seed_rows_settled: list[int] = []  # KB rows of seeds the next in-batch route() would have settled
    last_seeds: list = []              # seeds of the final query stay pending (router.py:333-334)
    cnt = {L: [0, 0] for L in LayerTag}  # probes, hits
    for j in range(p):
        q, L, probes = qs[j], serving[j], probes_all[j]
        for pr in probes:
            cnt[pr.layer][0] += 1
            cnt[pr.layer][1] += pr.outcome == "hit"
        seeds = ()
        lat = router.latency_model.sample(L) if synthetic else wall / max(1, p)
        if L is L1 or L is L2:
            if L is L1:
                a = latest.get(q.text) or kv.entry_at(int(kv_val[j])).answer
            else:
                t = sc_index.id_at(int(sc_row[j]))
                a = latest.get(t) or sc_index.payload_at(int(sc_row[j])).answer
            # served_as(L, 0.0) then answer_with_latency (model.py:177-192): a
            # cache-served copy of a validated record, passages dropped
            ans = AnswerRecord._trusted(a.text, L, a.confidence, (), lat)
        elif L is L3:
            a = recalled[j]
            ans = AnswerRecord._trusted(a.text, L, a.confidence, (), lat)
        else:
            s = slot[j]
            rows = kb_rows[s, : kb_cnt[s]]
            seeds = [kb.index.payload_at(int(r)) for r in rows]
            a = generation.generate_with_context(backend, q, seeds[: cfg.retrieval_k], L5)
            ans = AnswerRecord._trusted(a.text, L5, a.confidence, a.supporting_passage_ids, lat)
            if j < p - 1:
                seed_rows_settled.extend(int(r) for r in rows)
            else:
                last_seeds = seeds
        if synthetic:
            probes[-1] = LayerProbe(probes[-1].layer, probes[-1].outcome, lat)
        latest[q.text] = ans
        answers.append(ans)
        events.append(RouteTraceEvent(q.id, q.session_id, q.text, tuple(probes), L, lat, q.issued_at, ans.text,
                                      router._passage_pairs(ans, seeds)))

    prof.mark("materialise")
    # write-back (router.py:333-337): KV in order (last write wins), SC rows/payloads
    kv.put_many(texts[:p], answers)
    n_new_kept = int(np.searchsorted(new_js, p, side="left"))
    if n_pre_sc + n_new_kept < len(sc_index):
        sc_index.truncate(n_pre_sc + n_new_kept)
    now = time.monotonic_ns()
    with sc._lock:
        for j in range(p):
            t = texts[j]
            row = sc_index.row_of(t)
            sc_index._payloads[row] = CacheEntry(query_text=t, answer=answers[j], created_at_ns=now)
            sc._seq += 1
            sc._recency[t] = sc._seq
    # AKM: seeds of queries before the last were settled by the following
    # route() calls (device-to-device from KB rows, dedupe by id, no overwrite);
    # the last query's seeds are still pending, exactly as after route()
    if seed_rows_settled:
        akm.settle_from_rows(kb.index, seed_rows_settled)
    if last_seeds:
        akm.enqueue(last_seeds)

    # counters
    kv.hits += cnt[L1][1]
    kv.misses += cnt[L1][0] - cnt[L1][1]
    sc.hits += cnt[L2][1]
    sc.misses += cnt[L2][0] - cnt[L2][1]
    sc_index.search_count += cnt[L2][0]
    akm.misses += cnt[L4][0]
    akm.index.search_count += cnt[L4][0]
    kb.index.search_count += cnt[L5][0]
    router.trace.extend(events)
    prof.mark("writeback")
    if prof.enabled:
        hist = getattr(router, "batch_profile", None)
        if hist is None:
            hist = router.batch_profile = {}
        for k, v in prof.times.items():
            hist[k] = hist.get(k, 0.0) + v
    return p, list(zip(answers, events))


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

    def mark(self, name: str) -> None:
        if not self.enabled:
            return
        import torch

        torch.cuda.synchronize()
        t = time.perf_counter()
        self.times[name] = self.times.get(name, 0.0) + (t - self._t)
        self._t = t
