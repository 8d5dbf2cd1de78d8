"""Isolate the bench-vs-probe C5 slowdown: store from bench.build_shard, optional
headline-like searches first (HEADLINE=1)."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from benchlib import configs as C  # noqa: E402

n = 10_000_000
idx = bench.build_shard(n, 1024, 0, n)
if os.environ.get("HEADLINE"):
    from paper_2506_21593_b200.sharded import ShardedFlatIndex

    q = bench.make_queries(n, 1024, 4096)
    sh = ShardedFlatIndex(idx, 0)
    for _ in range(8):
        sh.search_batch(q, 5)
    torch.cuda.synchronize()
r = C.c5_routed(idx, n, n_sessions=2, queries_per_session=20000, profile=True)
print(int(r["value"]), {k: round(v, 3) for k, v in r["stage_seconds"].items()
                        if k.split(".")[0] in ("sc", "kb", "seeds", "akm") and not k.endswith(("rows", "collected", "tensor_path"))})
