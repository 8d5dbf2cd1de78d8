"""Per-call time of small-store searches (the routed replay's cache/AKM/seed stores)."""
from __future__ import annotations

import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2506_21593_b200 import MODE_EXACT, MODE_TENSOR, MODE_TENSOR_I8  # noqa: E402
from scripts.probe_perf import make_queries, make_store  # noqa: E402

for case in os.environ.get("CASES", "40000x1024x2048x1,40000x1024x2048x10,200000x1024x2048x1").split(","):
    n, d, b, k = (int(x) for x in case.split("x"))
    idx = make_store(n, d)
    q = make_queries(idx, b, d)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, mode in (("i8", MODE_TENSOR_I8), ("fp16", MODE_TENSOR), ("exact", MODE_EXACT)):
        ts = []
        for r in range(12):
            torch.cuda.synchronize()
            s.record()
            idx.search_batch(q, k, mode=mode, validate=False)
            e.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(s.elapsed_time(e))
        st = idx.stats()
        print(f"{case} {name:5s}: median {statistics.median(ts):7.3f} ms  min {min(ts):7.3f}  max {max(ts):7.3f}  "
              f"appended={st.appended} rescored={st.candidates} fallback={st.fallback}", flush=True)
    del idx, q
    torch.cuda.empty_cache()
