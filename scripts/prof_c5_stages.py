"""C5 host path over a 2M-row KB (host-bound: the L5 scan is small), one 111k-query session:
routed q/s with the span stage timer off, then per-stage host ms per 4096-query span with it on,
then a cProfile of the finish stage's top functions."""
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
qps = int(os.environ.get("C5_QPS", 111112))
idx = bench.build_shard(n, 1024, 0, n)
torch.cuda.synchronize()


def run(profile=False):
    return C.c5_routed(idx, n, n_sessions=1, queries_per_session=qps, parity_queries=0, l5_oracle_queries=0,
                       profile=profile)


for i in range(2):
    r = run()
    print("plain", i, round(r["value"]), "routed q/s", flush=True)
r = run(profile=True)
st = r.get("stage_seconds") or {}
spans = max(1, -(-qps // 4096))
print("profiled", round(r["value"]), "routed q/s; ms per span by stage:")
for k, v in sorted(st.items(), key=lambda kv: -kv[1]):
    print(f"  {k:14s} {v * 1e3 / spans:7.2f}")
if os.environ.get("C5_CPROFILE", "1") == "1":
    pr = cProfile.Profile()
    pr.enable()
    r = run()
    pr.disable()
    print("cprofile run", round(r["value"]))
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats("paper_2506|_lib|pinned|ledger", 45)
    print(s.getvalue()[:12000])
