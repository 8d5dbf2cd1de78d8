"""TEST INFRASTRUCTURE ONLY — drives the REAL reference router for BASELINE configs[0] (C1).

C1 = the reference CPU PentaRAG router on a synthetic TriviaQA-style stream: Q/A pool
``synthetic_qa_dataset(100_000, seed=42)[:10_000]``, KB = ``dataset_to_corpus`` of all
100k rows (100k chunks), dim 384, ``SimulationConfig(n_sessions=9, queries_per_session=1000,
seed=0)``.  The reference is hard-wired to dim 1024; the shim
below sets ``ragcascade.embedding.DIMENSION`` (read at call time by ``EmbeddingVector.wrap``
and ``HashEmbedder``, embedding.py:30,56-59,146-157) and re-binds the three ``dim=DIMENSION``
defaults frozen at import (index.py:76, knowledge.py:44,170).

Two drivers:

* ``run_reference_simulation`` calls the reference's own ``run_simulation``
  (simulation.py:268-314) — the golden generator uses it.
* ``run_reference_session`` runs ONE session exactly as ``run_simulation``'s loop body does
  for session ``s`` (simulation.py:290-313); sessions are independent because
  ``reset_session()`` clears both caches and the AKM (router.py:366-372) and every RNG is
  seeded by ``[seed, s, …]`` — SPEC.md:640's "independent sessions" axis.  The bench's
  9-process CPU baseline runs one session per process with it; a CPU test checks it gives
  the same lines as ``run_simulation``.

Only tests/, tests/golden/ and bench.py's reference/cpu_baseline legs import this module.
"""
from __future__ import annotations

import json
import os
import sys
import time

C1_DIM = 384
C1_KB_ROWS = 100_000
C1_QA_ROWS = 10_000
C1_SESSIONS = 9
C1_QUERIES = 1000
C1_SEED = 0
C1_DATASET_SEED = 42

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
REF_PATHS = (os.path.join(_ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def load_reference():
    """Import ``ragcascade`` from the offline install (baseline/_ref) or the read-only source tree."""
    if "ragcascade" in sys.modules:
        return sys.modules["ragcascade"]
    for p in REF_PATHS:
        if os.path.isdir(os.path.join(p, "ragcascade")):
            sys.path.insert(0, p)
            try:
                import ragcascade
            finally:
                sys.path.remove(p)
            return ragcascade
    raise ImportError("reference ragcascade not found (baseline/_ref or /root/reference/pkg/src)")


def shim_dim(rc, dim: int) -> None:
    """Re-point the reference's hard-wired 1024 at ``dim``."""
    import ragcascade.embedding as E
    import ragcascade.index as I
    import ragcascade.knowledge as K

    E.DIMENSION = dim
    if hasattr(I, "DIMENSION"):
        I.DIMENSION = dim
    I.FlatIndex.__init__.__defaults__ = (dim,)
    K.MainKnowledgeBase.__init__.__defaults__ = (dim, "corpus")
    d = list(K.AdaptiveKnowledgeMemory.__init__.__defaults__)
    d[0] = dim
    K.AdaptiveKnowledgeMemory.__init__.__defaults__ = tuple(d)


def c1_rows(rc, n: int = C1_KB_ROWS):
    from ragcascade.datagen import synthetic_qa_dataset

    return synthetic_qa_dataset(n, seed=C1_DATASET_SEED)


def build_reference_router(rc, rows, dim: int = C1_DIM):
    """KB = dataset_to_corpus(rows) ingested with the reference HashEmbedder (knowledge.py:118-157)."""
    from ragcascade.simulation import dataset_to_corpus

    shim_dim(rc, dim)
    emb = rc.HashEmbedder()
    kb = rc.MainKnowledgeBase()
    rc.ingest_corpus((json.dumps(r) for r in dataset_to_corpus(rows)), emb, kb=kb)
    return rc.CascadeRouter(embedder=emb, backend=rc.StubBackend(), knowledge_base=kb)


def run_reference_simulation(rc, router, qa_rows, n_sessions=C1_SESSIONS, n_queries=C1_QUERIES, seed=C1_SEED):
    logs = rc.run_simulation(rc.SimulationConfig(n_sessions=n_sessions, queries_per_session=n_queries, seed=seed),
                             router, qa_rows)
    return [list(log.to_jsonl_lines()) for log in logs]


def run_reference_session(rc, router, qa_rows, s: int, n_queries=C1_QUERIES, seed=C1_SEED, sigma=None):
    """Session ``s`` of ``run_simulation`` alone (simulation.py:290-313).  Returns (lines, seconds)."""
    import numpy as np
    from ragcascade.metrics import LayerCostModel, SyntheticLatencyModel
    from ragcascade.simulation import RAMPS, SessionLog, SessionState, SimClock, SimulationConfig, next_query

    cfg = SimulationConfig(n_sessions=s + 1, queries_per_session=n_queries, seed=seed)
    if router.latency_model is None:
        router.latency_model = SyntheticLatencyModel(LayerCostModel(), sigma=cfg.latency_sigma)
    questions = [str(r["question"]) for r in qa_rows]
    t0 = time.perf_counter()
    router.reset_session()
    rng = np.random.default_rng([cfg.seed, s, 0])
    if hasattr(router.latency_model, "reseed"):
        router.latency_model.reseed([cfg.seed, s, 1])
    clock = SimClock()
    router.clock_ns = clock.now_ns
    state = SessionState(session_id=f"session_{s:02d}", questions=questions, queries_per_session=n_queries,
                         ramp=RAMPS[cfg.ramp], replay_split=cfg.replay_split, clock=clock)
    log = SessionLog(session_id=state.session_id)
    for _ in range(n_queries):
        query, origin = next_query(state, rng)
        answer, event = router.route(query)
        clock.advance(answer.latency_seconds)
        state.record_issued(query.text)
        log.events.append(event)
        log.origins.append(origin)
    return list(log.to_jsonl_lines()), time.perf_counter() - t0


def _session_worker(args):
    s, n_queries, kb_rows, dim = args
    rc = load_reference()
    rows = c1_rows(rc, kb_rows)
    router = build_reference_router(rc, rows, dim)
    lines, secs = run_reference_session(rc, router, rows[:C1_QA_ROWS], s, n_queries)
    return s, lines, secs


def run_sessions_parallel(sessions, n_queries=C1_QUERIES, kb_rows=C1_KB_ROWS, dim=C1_DIM, procs=None):
    """One process per session (mode ii of BASELINE.md §3).  Returns ({s: lines}, {s: seconds}, wall)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(procs or len(sessions)) as pool:
        out = pool.map(_session_worker, [(s, n_queries, kb_rows, dim) for s in sessions])
    wall = time.perf_counter() - t0
    return {s: l for s, l, _ in out}, {s: t for s, _, t in out}, wall
