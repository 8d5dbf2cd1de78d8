"""C5 alone: the bench's 10M x 1024 store, then benchlib.configs.c5_routed (env: C5_SESSIONS,
C5_QUERIES, C5_PROFILE=1, C5_PARITY=queries checked against the reference router, C5_BATCH=span,
C5_WORKERS=concurrent session replays)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from benchlib import configs as C  # noqa: E402

n = int(os.environ.get("C5_ROWS", 10_000_000))
idx = bench.build_shard(n, 1024, 0, n)
torch.cuda.synchronize()
r = C.c5_routed(idx, n, n_sessions=int(os.environ.get("C5_SESSIONS", 4)),
                queries_per_session=int(os.environ.get("C5_QUERIES", 20000)),
                profile=bool(os.environ.get("C5_PROFILE")), parity_queries=int(os.environ.get("C5_PARITY", 1000)),
                batch=int(os.environ.get("C5_BATCH", 4096)), workers=int(os.environ.get("C5_WORKERS", 1)))
print(json.dumps(r))
