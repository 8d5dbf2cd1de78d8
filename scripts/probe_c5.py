"""Stage profile of the routed C5 replay (route_batch) over an n-row store."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from benchlib import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--queries", type=int, default=8000)
ap.add_argument("--sessions", type=int, default=1)
a = ap.parse_args()
torch.cuda.set_device(0)
idx = bench.build_shard(a.n, 1024, 0, a.n)
r = C.c5_routed(idx, a.n, n_sessions=a.sessions, queries_per_session=a.queries, profile=True, parity_queries=50)
print(json.dumps(r, indent=1))
