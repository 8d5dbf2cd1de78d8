"""cProfile of the C5 routed replay's timed loop (host hotspots)."""
from __future__ import annotations

import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from benchlib import configs as C  # noqa: E402
from scripts.probe_perf import make_store  # noqa: E402

n = int(os.environ.get("N", "10000000"))
store = make_store(n, 1024)
pr = cProfile.Profile()
pr.enable()
r = C.c5_routed(store, n, n_sessions=2, queries_per_session=20000, parity_queries=0)
pr.disable()
print("value", r["value"])
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(45)
st.sort_stats("tottime").print_stats(30)
