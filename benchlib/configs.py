"""Secondary BASELINE.json configurations measured inside bench.py (rank 0, N=1).

C2  semantic-cache top-1 + threshold 0.85 over 1M x 768, batch 4096
C3  fixed-KV exact lookup, 100M keys, batch 65536 (fused fingerprint + probe)
C5  routed replay through all five layers over the 10M x 1024 store (LLM stubbed):
    nine-session-style warm-up sessions routed with route_batch

Each returns a dict that bench.py nests under "configs"; every number is
device-timed with CUDA events and comes with its own parity check.
"""
from __future__ import annotations

import gc
import os
import time

import numpy as np


def _events():
    import torch

    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _unit_rows(n, d, seed, device="cuda"):
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    x = torch.randn((n, d), generator=g, device=device, dtype=torch.float64)
    return (x / x.norm(dim=1, keepdim=True)).float()


# ---------------------------------------------------------------- C2
def c2_semantic(peak_tops: float, peak_how: str = "", p8=None, n=1_000_000, d=768, batch=4096, steps=20, threshold=0.85,
                parity_q=64):
    import torch

    from oracle import flat_index as F
    from paper_2506_21593_b200 import FlatIndex, HashEmbedder, SemanticCache

    sc = SemanticCache(HashEmbedder(dim=d), threshold=threshold, dim=d)
    X = _unit_rows(n, d, 21)
    sc.index.extend_arrays([f"t{i}" for i in range(n)], X, validate=False)
    g = torch.Generator(device="cuda").manual_seed(22)
    B2 = batch // 2
    # half: perturbed copies of stored rows with cosine ~ U(0.80, 0.99); half: fresh random
    rows = torch.randint(0, n, (B2,), generator=g, device="cuda")
    base = X[rows].double()
    noise = torch.randn((B2, d), generator=g, device="cuda", dtype=torch.float64)
    noise = noise - (noise * base).sum(1, keepdim=True) * base
    noise = noise / noise.norm(dim=1, keepdim=True)
    cos = 0.80 + 0.19 * torch.rand((B2, 1), generator=g, device="cuda", dtype=torch.float64)
    near = cos * base + (1 - cos ** 2).sqrt() * noise
    Q = torch.cat([near, _unit_rows(batch - B2, d, 23).double()])
    Q = (Q / Q.norm(dim=1, keepdim=True)).float().contiguous()
    for _ in range(3):
        sc.lookup_batch(Q, account=False)
    sc.index.set_timing(True)
    sc.index.scan_time()
    torch.cuda.synchronize()
    e0, e1 = _events()
    e0.record()
    for _ in range(steps):
        hit, row, score = sc.lookup_batch(Q, account=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    kms, kn = sc.index.scan_time()
    sc.index.set_timing(False)
    kern = kms / max(1, kn)
    flop = 2.0 * n * d * batch
    # parity: exact top-1 + threshold decision vs the oracle on sampled queries
    sel = np.r_[0:parity_q // 2, batch - parity_q // 2:batch]
    want = F.c_search(X.cpu().numpy(), Q[torch.from_numpy(sel).cuda()].cpu().numpy(), 1)
    got_hit = hit.cpu().numpy()[sel]
    got_row = row.cpu().numpy()[sel]
    want_hit = (want.count > 0) & (want.reported[:, 0] >= threshold)
    mism = int(((got_hit != want_hit) | (want_hit & (got_row != want.rows[:, 0]))).sum())
    probes = _c2_threshold_probes(sc, X, Q, B2, threshold, n_probe_queries=32)
    sc.threshold = threshold
    return {
        "workload": f"semantic-cache top-1 + threshold {threshold} over {n} x {d}, batch {batch} (configs[1])",
        "value": batch / (ms / 1e3), "unit": "lookups/s", "ms_per_batch": ms,
        "hit_fraction": float(hit.float().mean().item()),
        "roofline": {"bound": "tensor", "achieved": flop / (kern / 1e3) / 1e12, "peak": peak_tops,
                     "unit": "TOP/s", "frac": flop / (kern / 1e3) / 1e12 / peak_tops, "kernel_ms": kern,
                     "kernel": "tc8_scan_kernel", "peak_kind": peak_how,
                     "frac_of_inrun_cublas_int8": (flop / (kern / 1e3) / 1e12 / p8["int8_tops_sustained"]
                                                   if p8 else None)},
        "parity": {"queries_checked": int(sel.size), "mismatches": mism},
        "threshold_probes": probes,
    }


def _c2_threshold_probes(sc, X, Q, n_near, threshold, n_probe_queries=32):
    """64 threshold-boundary probes at 1M x 768 (the reference's
    equality/nextafter acceptance test, tests/test_acceptance.py:142-182, at scale).
    For 32 near-duplicate queries the oracle (C einsum restatement over all 1M rows) gives
    the exact reported top-1 score s; the cache is then asked with threshold = s (the
    inclusive gate, caches.py:140, must HIT) and threshold = nextafter(s, +inf) (must MISS),
    and the served row and score bits must equal the oracle's."""
    import torch

    from oracle import flat_index as F

    sel = np.linspace(0, n_near - 1, n_probe_queries).astype(np.int64)
    Qs = Q[torch.from_numpy(sel).cuda()]
    want = F.c_search(X.cpu().numpy(), Qs.cpu().numpy(), 1)
    bad, probes, skipped = 0, 0, 0
    for j in range(sel.size):
        s = float(want.reported[j, 0])
        if not (0.0 < s < 1.0):
            skipped += 1
            continue
        for thr, expect in ((s, True), (float(np.nextafter(s, np.inf)), False)):
            sc.threshold = thr
            hit, row, score = sc.lookup_batch(Qs[j:j + 1], account=False)
            probes += 1
            # a hit serves the exact top-1 (row and score bits); a miss is a miss
            ok = bool(hit.item()) == expect and (not expect or (int(row.item()) == int(want.rows[j, 0])
                                                               and float(score.item()) == s))
            bad += 0 if ok else 1
    return {"probes": probes, "mismatches": bad, "skipped_queries": skipped,
            "oracle": "oracle/einsum_order.c over all rows; threshold = exact top-1 score (hit) and its nextafter (miss)"}


# ---------------------------------------------------------------- C4 batch sweep
def c4_batch_sweep(idx, make_queries, n: int, d: int, batches=(256, 1024, 8192), k=5, warmup=3, steps=5):
    """The headline search (top-5 over the n x d store) at other batch sizes (SURVEY §8d
    C4: sweep 256..16384); each step is one search_batch over queries already in HBM,
    the store (10 GB of int8) is far larger than L2."""
    import torch

    out = {"workload": f"top-{k} over the {n} x {d} bench store, batch sweep (configs[3] shape, 1 GPU)",
           "unit": "queries/s", "points": []}
    for B in batches:
        q = make_queries(n, d, B)
        for _ in range(warmup):
            idx.search_batch(q, k, validate=False, count=False)
        torch.cuda.synchronize()
        e0, e1 = _events()
        e0.record()
        for _ in range(steps):
            idx.search_batch(q, k, validate=False, count=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        st = idx.stats()
        out["points"].append({"batch": B, "value": B / (ms / 1e3), "ms_per_step": ms, "path": int(st.path),
                              "fallback_queries": int(st.fallback)})
        del q
    return out


# ---------------------------------------------------------------- C3
def _key_arena(ids: np.ndarray):
    """'query-%09d' (or wider) keys as a UTF-8 arena + offsets, built with numpy."""
    digits = np.maximum(9, np.floor(np.log10(np.maximum(ids, 1))).astype(np.int64) + 1)
    lens = 6 + digits
    off = np.zeros(ids.size + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    buf = np.empty(int(off[-1]), dtype=np.uint8)
    prefix = np.frombuffer(b"query-", dtype=np.uint8)
    for L in np.unique(lens):
        m = lens == L
        sub = ids[m]
        nd = int(L) - 6
        block = np.empty((sub.size, int(L)), dtype=np.uint8)
        block[:, :6] = prefix
        v = sub.copy()
        for c in range(nd - 1, -1, -1):
            block[:, 6 + c] = 48 + (v % 10)
            v //= 10
        starts = off[:-1][m]
        idx = (starts[:, None] + np.arange(int(L))[None, :]).ravel()
        buf[idx] = block.ravel()
    return buf, off


def _kv_get(L, h, b, out, hit, stream):
    from paper_2506_21593_b200 import _lib

    L.pr_kv_get_text(h, _lib.ptr(b[0]), _lib.ptr(b[1]), b[1].shape[0] - 1, _lib.ptr(out),
                     _lib.ptr(hit), stream)


def c3_kv(hbm_gbs: float, n_keys=100_000_000, batch=65536, n_batches=32, steps=5, chunk=8_000_000, streams=8):
    """C3: byte-exact fixed-KV lookups (pr_kv_get_text: hash + probe + record confirm) over a
    100M-key table, batches of 65536.  The batch stream is replayed as one CUDA graph whose
    batches run on ``streams`` concurrent branches (independent request batches in flight at
    once, as a serving loop has them); the single-stream graph and the eager loop are
    reported beside it."""
    import ctypes

    import torch

    from paper_2506_21593_b200 import _lib

    L = _lib.load()
    h = ctypes.c_void_p()
    _lib.check(L.pr_kv_create(n_keys, ctypes.byref(h)))
    s = _lib.stream_ptr()
    t0 = time.time()
    for c0 in range(0, n_keys, chunk):
        ids = np.arange(c0, min(n_keys, c0 + chunk), dtype=np.int64)
        buf, off = _key_arena(ids)
        d_buf, d_off = torch.from_numpy(buf).cuda(), torch.from_numpy(off).cuda()
        vals = torch.from_numpy(ids).cuda()
        _lib.check(L.pr_kv_put_text(h, _lib.ptr(d_buf), _lib.ptr(d_off), ids.size, int(off[-1]), _lib.ptr(vals), s))
    torch.cuda.synchronize()
    build_s = time.time() - t0
    size = L.pr_kv_size(h, s)
    mem = [ctypes.c_int64() for _ in range(3)]
    _lib.check(L.pr_kv_memory(h, *(ctypes.byref(m) for m in mem), s))
    rng = np.random.default_rng(3)
    batches = []
    for _ in range(n_batches):
        present = rng.integers(0, n_keys, batch // 2)
        absent = rng.integers(n_keys, 2 * n_keys, batch - batch // 2)
        ids = np.concatenate([present, absent])
        rng.shuffle(ids)
        buf, off = _key_arena(ids)
        batches.append((torch.from_numpy(buf).cuda(), torch.from_numpy(off).cuda(), torch.from_numpy(ids).cuda()))
    outs = [(torch.empty(batch, dtype=torch.int64, device="cuda"), torch.empty(batch, dtype=torch.uint8, device="cuda"))
            for _ in range(n_batches)]
    for b, (o, hh) in zip(batches[:3], outs):
        _kv_get(L, h, b, o, hh, s)
    torch.cuda.synchronize()
    e0, e1 = _events()
    e0.record()
    for _ in range(steps):
        for b, (o, hh) in zip(batches, outs):
            _kv_get(L, h, b, o, hh, s)
    e1.record()
    torch.cuda.synchronize()
    ms_eager = e0.elapsed_time(e1)
    lookups = steps * n_batches * batch

    def graph_of(nstreams):
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        side = [torch.cuda.Stream() for _ in range(nstreams - 1)]
        with torch.cuda.stream(cap):
            with torch.cuda.graph(g, stream=cap):
                for st in side:  # fork
                    st.wait_stream(cap)
                branches = [cap] + side
                for i, (b, (o, hh)) in enumerate(zip(batches, outs)):
                    br = branches[i % nstreams]
                    _kv_get(L, h, b, o, hh, _lib.stream_ptr(br))
                for st in side:  # join
                    cap.wait_stream(st)
        torch.cuda.current_stream().wait_stream(cap)
        return g

    def time_graph(g):
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    ms_serial = time_graph(graph_of(1))
    ms = time_graph(graph_of(streams))
    # parity: every lookup of every batch against the construction (value = key id, absent -> -1)
    bad = 0
    for b, (o, hh) in zip(batches, outs):
        want = torch.where(b[2] < n_keys, b[2], torch.full_like(b[2], -1))
        bad += int(((o != want) | (hh.bool() != (b[2] < n_keys))).sum().item())
    # the same probe on one large batch (4M keys): the throughput-bound regime of the kernel
    big_ids = np.concatenate([rng.integers(0, n_keys, 2 << 20), rng.integers(n_keys, 2 * n_keys, 2 << 20)])
    bbuf, boff = _key_arena(big_ids)
    big = (torch.from_numpy(bbuf).cuda(), torch.from_numpy(boff).cuda())
    bout = torch.empty(big_ids.size, dtype=torch.int64, device="cuda")
    bhit = torch.empty(big_ids.size, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        _kv_get(L, h, big, bout, bhit, s)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        _kv_get(L, h, big, bout, bhit, s)
    e1.record()
    torch.cuda.synchronize()
    big_ms = e0.elapsed_time(e1) / 5
    want_big = torch.from_numpy(np.where(big_ids < n_keys, big_ids, -1)).cuda()
    bad += int((bout != want_big).sum().item())
    L.pr_kv_destroy(h)
    per_s = lookups / (ms / 1e3)
    gbs = per_s * 56 / 1e9
    big_per_s = big_ids.size / (big_ms / 1e3)
    return {
        "workload": f"fixed-KV byte-exact lookup, {n_keys} keys, batch {batch}, 50% present (configs[2], 1 GPU)",
        "value": per_s, "unit": "lookups/s", "us_per_batch": ms * 1e3 / (steps * n_batches),
        "launch": f"{n_batches} batches per CUDA graph replay on {streams} concurrent graph branches "
                  "(one pr_kv_get_text kernel per 65536-key batch)",
        "serial_graph": {"value": lookups / (ms_serial / 1e3), "us_per_batch": ms_serial * 1e3 / (steps * n_batches),
                         "launch": "same graph, one branch (batches back to back)"},
        "eager": {"value": lookups / (ms_eager / 1e3), "us_per_batch": ms_eager * 1e3 / (steps * n_batches),
                  "launch": "one ctypes pr_kv_get_text call per batch from Python"},
        "keys_live": int(size), "build_seconds": build_s,
        "table_bytes": {"slots": mem[0].value, "records": mem[1].value, "garbage": mem[2].value},
        "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_gbs, "unit": "GB/s", "frac": gbs / hbm_gbs,
                     "bytes_per_lookup": 56,
                     "note": "algorithmic 56 B per lookup (16-B key + one 32-B table sector + 8-B value, SURVEY "
                             "§8d); the kernel also confirms every tag match against the stored key bytes",
                     # what the DRAM actually charges: one random 128-B line per lookup (+ key, offsets,
                     # outputs) — ncu 156 B read + 9 B written per lookup (profiles/r02c_kv_get_ncu_summary.txt);
                     # the random-line ceiling of this part is ~45.3 G lines/s (scripts/micro/randline.cu,
                     # profiles/r02_kv_layout_experiments.txt)
                     "physical": {"dram_bytes_per_lookup": 165, "achieved_GBps": per_s * 165 / 1e9,
                                  "frac_of_hbm": per_s * 165 / 1e9 / hbm_gbs,
                                  "random_line_ceiling_per_s": 45.3e9,
                                  "frac_of_random_line_ceiling": per_s / 45.3e9,
                                  "source": "ncu dram bytes per lookup (r02c capture) and the randline micro; "
                                            "constants, not measured in this run"}},
        "large_batch": {"batch": int(big_ids.size), "value": big_per_s, "unit": "lookups/s",
                        "algorithmic_GBps": big_per_s * 56 / 1e9, "frac_of_hbm": big_per_s * 56 / 1e9 / hbm_gbs},
        "parity": {"lookups_checked": n_batches * batch + int(big_ids.size), "mismatches": bad},
    }


# ---------------------------------------------------------------- C5
class _RowVector:
    """Passage.embedding of a dense distractor row, read from the device store on demand."""

    def __init__(self, store, row):
        self._store, self._row = store, row

    @property
    def values(self):
        return self._store.read_rows(self._row, 1).cpu().numpy()[0]


class _KBPayloads:
    """Payload list of the 10M-row bench KB: real Passages for the QA contexts,
    distractor Passages (own id, own stored vector) materialised on access."""

    def __init__(self, store, real):
        from paper_2506_21593_b200 import Passage

        self._store, self._real, self._n = store, real, len(store._ids)
        self._n_real, self._passage = len(real), Passage

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if i < self._n_real:
            return self._real[i]
        return self._passage(id=self._store.id_at(i), text=f"Distractor passage {i}. Unrelated archival material.",
                       source="distractor", embedding=_RowVector(self._store, i), answer=None)


_LAST_PROFILE_LOG: list = []  # per-batch stage times of the last profiled c5_routed run
_LAST_BATCH_WALL: list = []  # (worker, session, batch, host wall ms) of every c5_routed batch


def c5_routed(store, n_store: int, *, n_qa=120_000, n_sessions=2, queries_per_session=20_000, batch=4096,
              seed=0, parity_queries=1000, profile=False, workers=1, l5_oracle_queries=8, shard=None,
              session_ids=None, group=None):
    """Routed replay over the bench's 10M x 1024 store turned into a knowledge base:
    rows [0, n_qa) hold HashEmbedder(context) of the QA pool, the rest stay dense
    distractors.

    ``workers`` > 1: that many routers (each its own KV / semantic cache / AKM, one
    shared knowledge base) replay the sessions concurrently from as many threads —
    sessions are independent, and one worker's host-side Python then
    overlaps another's device scans on the shared GPU.

    ``session_ids``: replay only these of the ``n_sessions`` sessions (multi-GPU session
    replicas: rank r of N routes sessions r, r+N, ... over its own full knowledge base).
    ``group``: the process group a row-sharded knowledge base (``shard``) spans (default: all
    ranks) — the hybrid layout: groups of ranks, each with its own sharded KB and sessions."""
    import threading

    import torch

    from benchlib.workloads import LatencyDraws, corpus_of, qa_rows, session_stream
    from paper_2506_21593_b200 import (CascadeRouter, HashEmbedder, LayerTag, MainKnowledgeBase, Passage,
                                       StubBackend, validate_query)
    from paper_2506_21593_b200.vectors import EmbeddingVector

    emb = HashEmbedder()
    t0 = time.time()
    rows = qa_rows(n_qa, seed=42)
    corpus = corpus_of(rows)
    ctx = emb.embed_matrix([c["text"] for c in corpus])
    if shard is None:
        store._update_rows(np.arange(n_qa, dtype=np.int64), ctx)
    else:
        # row-sharded knowledge base (multi-GPU): ``store`` is this rank's block of global rows
        # [row0, row0 + len(store)); the contexts' rows are updated where they live, and the
        # KB the routers see is the sharded view (sharded.ShardedRowIndex)
        from paper_2506_21593_b200.sharded import ShardedRowIndex

        row0 = int(shard)
        a, b = row0, min(row0 + len(store), n_qa)
        if a < b:
            store._update_rows(np.arange(a, b, dtype=np.int64) - row0, ctx[a:b])
        store = ShardedRowIndex.wrap(store, [str(i) for i in range(n_store)], None, row0, group=group)
        parity_queries = min(parity_queries, 200)
        l5_oracle_queries = 0
        workers = 1
    real = [Passage(id=store.id_at(i), text=c["text"], source=c["source"],
                    embedding=EmbeddingVector(values=ctx[i]), answer=c["answer"]) for i, c in enumerate(corpus)]
    store._payloads = _KBPayloads(store, real)
    kb = MainKnowledgeBase.from_index(store)
    questions = [r["question"] for r in rows]
    streams = [session_stream(questions, queries_per_session, seed, s) for s in range(n_sessions)]
    prep_s = time.time() - t0

    def make_router():
        r = CascadeRouter(embedder=emb, backend=StubBackend(), knowledge_base=kb)
        r.latency_model = LatencyDraws(0.25)
        return r

    workers = max(1, min(int(workers), n_sessions if session_ids is None else max(1, len(list(session_ids)))))
    routers = [make_router() for _ in range(workers)]
    # warm-up: one whole session of an unrelated seed per router, untimed (first-launch
    # module loading; the stores and search scratch grow to their per-session size, and
    # reset_session keeps that capacity, as in a serving process past its first session)
    _, warm = session_stream(questions, queries_per_session, seed + 1000, 0)
    wq = [validate_query(t, "warmup", query_id=f"w{i}", issued_at_ns=0) for i, (t, _) in enumerate(warm)]
    for router in routers:
        router.route_batch(wq, materialize=False, span=batch)
        router.reset_session()
        router.trace.clear()
        router.profile_batches = profile
    router = routers[0]
    # the sessions' validated Query objects are the router's input (built by the caller,
    # src/simulation.py:241-265 via validate_query), made before the timed region
    session_queries = [[validate_query(t, sid, query_id=f"{sid}-q{i:05d}", issued_at_ns=0) for i, (t, _) in enumerate(st)]
                       for sid, st in streams]
    # the loaded KB (10M ids, 120k passages) is permanent: keep it out of the cyclic
    # collector's full passes, which otherwise stall a batch for ~150 ms each
    # (measured, scripts/probe_growth.py) — standard practice for a loaded server;
    # the prepared session queries are frozen with it
    gc.collect()
    gc.freeze()
    tallies = [{"total": 0, "sequential": 0, "layers": {}} for _ in range(workers)]
    errors: list = []

    # one CUDA stream per worker: a worker's small kernels (embedding, probes, write-back)
    # need not queue behind another worker's knowledge-base scan (the shared KB handle
    # orders its own searches across streams)
    streams_w = [torch.cuda.current_stream()] if workers == 1 else [torch.cuda.Stream() for _ in range(workers)]
    for st_w in streams_w:
        st_w.wait_stream(torch.cuda.current_stream())

    def replay(w):
        try:
            with torch.cuda.stream(streams_w[w]):
                _replay_sessions(w, routers[w], tallies[w])
            streams_w[w].synchronize()
        except BaseException as exc:  # noqa: BLE001 - re-raised on the main thread
            errors.append(exc)

    mine_s = list(range(n_sessions)) if session_ids is None else [int(x) for x in session_ids]

    def _replay_sessions(w, router, tally):
        for s in mine_s[w::workers]:
            router.reset_session()
            router.latency_model.reseed([seed, s, 1])
            qs = session_queries[s]
            # ONE route_batch call per session: spans of `batch` queries, span i+1's device
            # stage queued before span i's host stage (cascade.py); columnar result (per-query
            # objects are only built if someone reads them); query texts in, embedded on the
            # device inside the call (pr_hash_embed)
            t_b = time.perf_counter()
            res = router.route_batch(qs, materialize=False, span=batch)
            st = router.last_batch_stats
            _LAST_BATCH_WALL.append((w, s, st["spans"], (time.perf_counter() - t_b) * 1e3 / max(1, st["spans"]),
                                     st["splits"]))
            tally["total"] += len(res)
            tally["sequential"] += st["sequential"]
            tally["spans"] = tally.get("spans", 0) + st["spans"]
            tally["pipelined"] = tally.get("pipelined", 0) + st["pipelined"]
            for code, c in zip(*np.unique(res.layers(), return_counts=True)):
                name = LayerTag(int(code)).wire_name
                tally["layers"][name] = tally["layers"].get(name, 0) + int(c)

    _LAST_BATCH_WALL.clear()
    gc_ms = [0.0, 0.0]  # total, longest collection inside the timed region

    def _gc_timer(phase, info, _t=[0.0]):
        if phase == "start":
            _t[0] = time.perf_counter()
        else:
            dt = (time.perf_counter() - _t[0]) * 1e3
            gc_ms[0] += dt
            gc_ms[1] = max(gc_ms[1], dt)

    gc.callbacks.append(_gc_timer)
    gc_stats0 = gc.get_stats()
    gc_off = os.environ.get("C5_GC_DISABLE") == "1"  # measurement knob: no cyclic GC while timed
    if gc_off:
        gc.disable()
    e0, e1 = _events()
    torch.cuda.synchronize()
    e0.record()
    torch.cuda.nvtx.range_push("c5_timed")  # ncu --nvtx-include c5_timed/ (launch lists of the replay only)
    if workers == 1:
        replay(0)
    else:
        pool = [threading.Thread(target=replay, args=(w,)) for w in range(workers)]
        for t in pool:
            t.start()
        for t in pool:
            t.join()
    for st_w in streams_w:
        torch.cuda.current_stream().wait_stream(st_w)
    e1.record()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if gc_off:
        gc.enable()
    gc.callbacks.remove(_gc_timer)
    gc_counts = [b["collections"] - a["collections"] for a, b in zip(gc_stats0, gc.get_stats())]
    walls = np.array([b[3] for b in _LAST_BATCH_WALL]) if _LAST_BATCH_WALL else np.zeros(1)
    if errors:
        raise errors[0]
    total = sum(t["total"] for t in tallies)
    seq_total = sum(t["sequential"] for t in tallies)
    layer_counts: dict = {}
    for t in tallies:
        for name, c in t["layers"].items():
            layer_counts[name] = layer_counts.get(name, 0) + c
    gc.unfreeze()
    # parity: the first parity_queries of session 0, routed by route_batch on a fresh router,
    # against the REAL reference router (ragcascade.CascadeRouter from the offline install in
    # baseline/_ref, router.py:275-364) driving fresh GPU stores over the same knowledge
    # base one query at a time; a twin of this package's route() when the install is absent
    sid, st = streams[0]
    qs = [validate_query(t, sid, query_id=f"{sid}-q{i:05d}", issued_at_ns=0) for i, (t, _) in enumerate(st)]
    qs = qs[:parity_queries]
    mine = make_router()
    mine.reset_session()
    mine.latency_model.reseed([seed, 0, 1])
    got = mine.route_batch(qs, span=256)  # several pipelined spans over the full-size KB
    mism, oracle_name = 0, "twin router, sequential route() per query (reference semantics)"
    try:
        from oracle.ref_c1 import load_reference

        rc = load_reference()
        from paper_2506_21593_b200 import AdaptiveKnowledgeMemory, FixedKVCache, SemanticCache

        rref = rc.CascadeRouter(embedder=rc.HashEmbedder(), backend=rc.StubBackend(), knowledge_base=kb,
                                kv_cache=FixedKVCache(), semantic_cache=SemanticCache(emb),
                                adaptive_memory=AdaptiveKnowledgeMemory())
        oracle_name = ("ragcascade.CascadeRouter (the reference, baseline/_ref) over GPU stores, one route() per "
                       "query: answers, serving layer, passages, per-layer probe outcomes")

        def ref_route(q):
            return rref.route(rc.validate_query(q.text, q.session_id))
    except ImportError:
        twin = make_router()
        twin.reset_session()
        twin.latency_model.reseed([seed, 0, 1])
        ref_route = twin.route
    l5_sample = []
    for q, (a, ev) in zip(qs, got):
        b, ev2 = ref_route(q)
        if (a.text, a.layer.wire_name, tuple(a.supporting_passage_ids),
            [(p.layer.wire_name, p.outcome) for p in ev.layers_probed]) != \
                (b.text, b.layer.wire_name, tuple(b.supporting_passage_ids),
                 [(p.layer.wire_name, p.outcome) for p in ev2.layers_probed]):
            mism += 1
        if a.layer == LayerTag.NAIVE_RAG and len(l5_sample) < l5_oracle_queries:
            l5_sample.append(q.text)
    l5 = _c5_l5_oracle(kb, emb, l5_sample) if l5_sample else None
    if profile:
        _LAST_PROFILE_LOG[:] = getattr(router, "batch_profile_log", [])
    return {
        "workload": f"five-layer routed replay (L1/L2/L3/L4/L5, LLM stubbed) over a {n_store} x 1024 KB "
                    f"({n_qa} HashEmbedder contexts + dense distractors), {n_sessions} cache-warming sessions x "
                    f"{queries_per_session} queries = {n_sessions * queries_per_session} routed queries, spans of "
                    f"{batch} (configs[4], {'1 GPU' if shard is None else 'KB row-sharded over all ranks'}), "
                    f"{workers} concurrent session worker(s)",
        "value": total / (ms / 1e3), "unit": "routed queries/s", "ms_total": ms, "workers": workers,
        "queries": total, "sessions": mine_s,
        "knowledge_base": ("one GPU" if shard is None else
                           f"row-sharded: this rank holds rows [{int(shard)}, {int(shard) + store.n_local}); local "
                           "list scan + one all-gather merge per span, seed/AKM rows gathered from their owners"),
        "layer_counts": layer_counts, "queries_routed_sequentially": seq_total,
        "spans": sum(t.get("spans", 0) for t in tallies), "spans_pipelined": sum(t.get("pipelined", 0) for t in tallies),
        "span_wall_ms_mean_per_session": {"n": int(walls.size), "median": float(np.median(walls)), "p90": float(np.percentile(walls, 90)),
                          "max": float(walls.max()), "sum": float(walls.sum())},
        "gc_ms_in_timed_region": {"total": gc_ms[0], "longest": gc_ms[1], "collections_per_generation": gc_counts,
                                  "disabled": gc_off},
        "stage_seconds": getattr(router, "batch_profile", None),
        "query_vectors": "device HashEmbedder (pr_hash_embed) inside the timed region, from raw query texts",
        "prep_seconds": prep_s,
        "parity": {"queries_checked": len(qs), "mismatches": mism, "oracle": oracle_name,
                   "l5_rows_vs_chunked_oracle": l5},
    }


def _c5_l5_oracle(kb, emb, texts, k=10, chunk=1 << 20):
    """Sampled L5 checks at full KB size: the knowledge-base top-k (seed_k) of each query
    from the GPU index vs the C einsum restatement streamed over all rows in 1M-row chunks
    (per-row scores are chunk-invariant), ranked by (score desc, row asc)."""
    from oracle import flat_index as F

    V = np.stack([emb.embed_array(t) for t in texts]).astype(np.float32)
    res = kb.index.search_batch(V, k, validate=False, count=False)
    rows, raw = res.rows.cpu().numpy(), res.raw.cpu().numpy()
    n = len(kb.index)
    cand_s, cand_r = [], []
    for r0 in range(0, n, chunk):
        m = min(chunk, n - r0)
        Xc = kb.index.read_rows(r0, m).cpu().numpy()
        o = F.c_search(Xc, V, k)
        cand_s.append(o.raw)
        cand_r.append(np.where(o.rows >= 0, o.rows + r0, -1))
    S, R = np.concatenate(cand_s, axis=1), np.concatenate(cand_r, axis=1)
    bad_rows = bad_scores = 0
    for q in range(len(texts)):
        ok = R[q] >= 0
        order = np.lexsort((R[q][ok], -S[q][ok]))[:k]
        wr, ws = R[q][ok][order], S[q][ok][order]
        bad_rows += int(not np.array_equal(wr, rows[q, :wr.size]))
        bad_scores += int(not np.array_equal(ws, raw[q, :ws.size]))
    return {"queries": len(texts), "k": k, "row_mismatches": bad_rows, "raw_score_mismatches": bad_scores}


def c1_routed(reference: bool = True, procs: int = 9, batch: int = 4096, reps: int = 3):
    """C1 (BASELINE configs[0]): the reference's nine-session cache-warming simulation —
    KB = dataset_to_corpus(synthetic_qa_dataset(100_000, 42)) at dim 384, Q/A pool = its first
    10k rows, SimulationConfig(9, 1000, seed=0) (simulation.py:268-314) — routed by
    ``route_batch`` over GPU stores.  ``value`` = routed queries/s of the whole simulation
    (``simulate_batched``: session logs materialised as JSONL, the reference's output),
    median of ``reps`` runs; parity = every session's lines byte-identical to the real
    reference's (fixture tests/golden/c1_sessions.json.gz, written by tests/golden/make_c1.py).

    ``reference``: the REAL reference router (baseline/_ref) on this host's cores, one process
    per session (sessions are independent; BASELINE.md §3 mode ii) — the C1
    CPU baseline; each process also checks its session's lines against the fixture."""
    import gzip
    import hashlib
    import json
    import os

    import torch

    from benchlib.workloads import corpus_of, qa_rows, simulate_batched
    from paper_2506_21593_b200 import CascadeRouter, HashEmbedder, StubBackend, ingest_corpus

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with gzip.open(os.path.join(root, "tests", "golden", "c1_sessions.json.gz"), "rt") as fh:
        fx = json.load(fh)
    cfg = fx["config"]
    t0 = time.perf_counter()
    rows = qa_rows(cfg["kb_rows"], seed=cfg["dataset_seed"])
    emb = HashEmbedder(dim=cfg["dim"])
    kb = ingest_corpus((json.dumps(c) for c in corpus_of(rows)), emb)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    questions = [r["question"] for r in rows[:cfg["qa_rows"]]]
    n_s, n_q = cfg["n_sessions"], cfg["queries_per_session"]
    router = CascadeRouter(embedder=emb, backend=StubBackend(), knowledge_base=kb)
    simulate_batched(router, questions, n_sessions=2, n_queries=n_q, seed=cfg["seed"] + 1000, batch=batch)  # warm-up
    times, logs = [], None
    for _ in range(reps):
        # the previous run's router (its stores hold device tables; reference cycles keep it
        # alive) is collected HERE, not by a GC pass inside the next timed run — destroying
        # a store synchronises the device and frees memory (two of three runs used to take 2x)
        del router
        gc.collect()
        torch.cuda.synchronize()
        router = CascadeRouter(embedder=emb, backend=StubBackend(), knowledge_base=kb)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        logs = simulate_batched(router, questions, n_sessions=n_s, n_queries=n_q, seed=cfg["seed"], batch=batch)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    digests = [hashlib.sha256("\n".join(s).encode()).hexdigest() for s in logs]
    sec = float(np.median(times))
    out = {
        "workload": f"C1 (configs[0]): reference nine-session cache-warming simulation, {cfg['kb_rows']} chunks x "
                    f"dim {cfg['dim']}, {n_s} sessions x {n_q} queries, route_batch spans of {batch} (1 GPU)",
        "value": n_s * n_q / sec, "unit": "routed queries/s", "seconds": sec, "runs": times,
        "timed": "simulate_batched: validate + route_batch + JSONL session logs, wall clock, after a warm-up",
        "kb_build_seconds": build_s,
        "layer_counts": {k: int(v) for k, v in router.stats()["layer_counts"].items() if v},
        "parity": {"sessions": n_s, "sessions_identical": int(sum(d == w for d, w in zip(digests, fx["sha256"]))),
                   "oracle": "real reference run_simulation session logs (sha256 per session, fixture)"},
    }
    if reference:
        try:
            from oracle import ref_c1 as R

            R.load_reference()
        except ImportError as exc:
            out["cpu_baseline"] = {"unavailable": f"reference not importable: {exc}"}
            return out
        sess = list(range(n_s))
        got, secs, wall = R.run_sessions_parallel(sess, n_q, procs=min(procs, n_s))
        route_max = max(secs.values())
        same = sum(hashlib.sha256("\n".join(got[s]).encode()).hexdigest() == fx["sha256"][s] for s in sess)
        out["cpu_baseline"] = {
            "value": n_s * n_q / route_max, "unit": "routed queries/s", "cores": min(procs, n_s), "kind": "reference",
            "sample": f"the full C1 simulation: {n_s} sessions, one process per session running the unmodified "
                      "reference router (baseline/_ref ragcascade, dim shim SURVEY §0.5); value = queries / the "
                      "slowest session's routing time (KB ingest per process not counted)",
            "route_seconds": {str(k): v for k, v in secs.items()}, "wall_seconds_incl_ingest": wall,
            "single_process_estimate": {"value": n_s * n_q / sum(secs.values()), "unit": "routed queries/s",
                                        "how": "queries / summed per-session routing time (mode i: one core)"},
            "sessions_identical_to_fixture": int(same),
        }
        out["speedup_vs_cpu_baseline"] = out["value"] / out["cpu_baseline"]["value"]
    return out
