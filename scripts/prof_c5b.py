"""cProfile of route_batch calls only (the C5 timed loop's host work)."""
from __future__ import annotations

import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from benchlib import configs as C  # noqa: E402
from paper_2506_21593_b200 import router as R  # noqa: E402
from scripts.probe_perf import make_store  # noqa: E402

pr = cProfile.Profile()
orig = R.CascadeRouter.route_batch


def rb(self, queries, vectors=None, **kw):
    pr.enable()
    try:
        return orig(self, queries, vectors=vectors, **kw)
    finally:
        pr.disable()


R.CascadeRouter.route_batch = rb
n = 10_000_000
store = make_store(n, 1024)
r = C.c5_routed(store, n, n_sessions=2, queries_per_session=20000, parity_queries=0,
                profile=bool(os.environ.get("STAGES")))
if os.environ.get("STAGES"):
    print({k: round(v, 4) for k, v in r["stage_seconds"].items() if "." not in k})
print("value", r["value"])
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(28)
