"""C5 routed-replay probe: stage timings and KB search stats per batch, for a
given search mode (PR_MODE env: auto|tensor|i8)."""
from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from benchlib import configs as C  # noqa: E402
from scripts.probe_perf import make_store  # noqa: E402


def main():
    mode = {"auto": 0, "tensor": 2, "i8": 3, "exact": 1}[os.environ.get("PR_MODE", "auto")]
    if mode:
        from paper_2506_21593_b200 import router as R

        orig = R.CascadeRouter.route_batch

        def rb(self, queries, vectors=None, **kw):
            kw.setdefault("mode", mode)
            return orig(self, queries, vectors=vectors, **kw)

        R.CascadeRouter.route_batch = rb
    n = int(os.environ.get("N", "10000000"))
    store = make_store(n, 1024)
    if os.environ.get("MARK_BATCHES"):
        from paper_2506_21593_b200 import router as R

        orig_rb = R.CascadeRouter.route_batch
        cnt = [0]

        def rb_marked(self, queries, vectors=None, **kw):
            print(f"--- batch {cnt[0]}", file=sys.stderr, flush=True)
            cnt[0] += 1
            return orig_rb(self, queries, vectors=vectors, **kw)

        R.CascadeRouter.route_batch = rb_marked
    import gc

    gc_log = []

    def _gc_cb(phase, info, _t=[0.0]):
        if phase == "start":
            _t[0] = time.perf_counter()
        elif (time.perf_counter() - _t[0]) > 0.005:
            gc_log.append((info["generation"], round((time.perf_counter() - _t[0]) * 1e3, 1)))

    gc.callbacks.append(_gc_cb)
    if os.environ.get("KB_STATS"):
        from paper_2506_21593_b200 import index as I

        orig_sb = I.FlatIndex.search_batch
        kb_log = []

        def sb(self, queries, k, **kw):
            if len(self) < 1_000_000:
                return orig_sb(self, queries, k, **kw)
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = orig_sb(self, queries, k, **kw)
            torch.cuda.synchronize()
            st = self.stats()
            kb_log.append((queries.shape[0], round((time.perf_counter() - t) * 1e3, 1), st.fallback, st.appended,
                           st.candidates))
            return r

        I.FlatIndex.search_batch = sb
    t0 = time.time()
    r = C.c5_routed(store, n, n_sessions=int(os.environ.get("S", "1")), queries_per_session=int(os.environ.get("Q", "12288")),
                    batch=int(os.environ.get("B", "4096")),
                    profile=not os.environ.get("C5_WORKERS"), workers=int(os.environ.get("C5_WORKERS", "1")))
    print({k: v for k, v in r.items() if k in ("value", "layer_counts", "stage_seconds", "parity", "queries_routed_sequentially")})
    print("gc pauses > 5 ms (generation, ms):", gc_log)
    if os.environ.get("KB_STATS"):
        print("kb searches (nq, ms, fallback, appended, rescored):", kb_log[:26])
    print("batch wall ms (worker, session, batch, ms, splits):",
          [(w, s, b, round(ms, 1), sp) for w, s, b, ms, sp in C._LAST_BATCH_WALL])
    log = C._LAST_PROFILE_LOG
    for i, t in enumerate(log):
        print(i, {k: round(v * 1e3, 1) for k, v in t.items() if "." not in k or k.startswith("wb.")})
    st = store.stats()
    print("last KB search: path", st.path, "fallback", st.fallback, "cand", st.candidates, "appended", st.appended,
          "queries", st.queries, "wall", round(time.time() - t0, 1))


if __name__ == "__main__" and not os.environ.get("KB_REPEAT"):
    main()


def kb_repeat(reps=12):
    """Repeated identical KB searches on C5-style (HashEmbedder) queries."""
    import numpy as np

    from benchlib import configs as C
    from benchlib.workloads import qa_rows, session_stream
    from paper_2506_21593_b200 import HashEmbedder

    n = int(os.environ.get("N", "10000000"))
    store = make_store(n, 1024)
    C.c5_routed(store, n, n_sessions=1, queries_per_session=4096)  # turns the store into the C5 KB
    emb = HashEmbedder()
    rows = qa_rows(120_000, seed=42)
    _, st = session_stream([r["question"] for r in rows], 4096, 5, 0)
    V = torch.from_numpy(np.stack([emb.embed(t).values for t, _ in st[:2048]])).cuda()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(reps):
        s.record()
        store.search_batch(V, 10, validate=False, count=False)
        e.record()
        torch.cuda.synchronize()
        stt = store.stats()
        print(f"rep {i}: {s.elapsed_time(e):.2f} ms appended={stt.appended} rescored={stt.candidates} "
              f"fallback={stt.fallback}", flush=True)


if __name__ == "__main__" and os.environ.get("KB_REPEAT"):
    kb_repeat()
