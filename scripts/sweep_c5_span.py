"""C5 span-size sweep on one store (bench's 10M x 1024): routed q/s per span size, same process and box."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from benchlib import configs as C  # noqa: E402

n = int(os.environ.get("C5_ROWS", 10_000_000))
idx = bench.build_shard(n, 1024, 0, n)
torch.cuda.synchronize()
for span in [int(x) for x in os.environ.get("C5_SPANS", "4096,8192,6144,4096,8192").split(",")]:
    r = C.c5_routed(idx, n, n_sessions=int(os.environ.get("C5_SESSIONS", 3)), queries_per_session=111112,
                    parity_queries=0, l5_oracle_queries=0, batch=span)
    print(span, round(r["value"]), "routed q/s; splits", r.get("spans"), r.get("queries_routed_sequentially"),
          "gc", round(r["gc_ms_in_timed_region"]["total"]), flush=True)
