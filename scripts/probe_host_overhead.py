"""Host-side cost of one search_batch call (no sync inside the timed call) per store
size / path: what a routed batch pays on the CPU for each device search it issues."""
from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from scripts.probe_perf import make_queries, make_store  # noqa: E402


def host_us(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t) * 1e6)
    torch.cuda.synchronize()
    return np.median(ts), min(ts)


for n, nq, k, lim in ((10_000_000, 3600, 10, False), (30_000, 3000, 1, True), (30_000, 3000, 1, False),
                      (3_000, 3000, 1, True)):
    idx = make_store(n, 1024)
    q = make_queries(idx, nq, 1024)
    rl = np.full(nq, n // 2, dtype=np.int64) if lim else None
    med, mn = host_us(lambda: idx.search_batch(q, k, validate=False, count=False, row_limit=rl))
    st = idx.stats()
    print(f"n={n} nq={nq} k={k} row_limit={lim}: host {med:.0f} us median ({mn:.0f} min), path {st.path}", flush=True)
    del idx
    torch.cuda.empty_cache()
