"""cProfile of the C5 host path (one 111k-query session over a 2M-row KB: the device part is
small, so the profile is the Python of route_batch's launch / finish stages)."""
import cProfile
import io
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from benchlib import configs as C  # noqa: E402

n = int(os.environ.get("C5_ROWS", 2_000_000))
idx = bench.build_shard(n, 1024, 0, n)
torch.cuda.synchronize()
pr = cProfile.Profile()
orig = C._LAST_BATCH_WALL


def run():
    return C.c5_routed(idx, n, n_sessions=1, queries_per_session=111112, parity_queries=0, l5_oracle_queries=0)


pr.enable()
r = run()
pr.disable()
print(r["value"], r["span_wall_ms_mean_per_session"])
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(30)
print(s.getvalue()[:7000])
