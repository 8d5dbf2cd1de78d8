"""A/B the tcgen05 scan schedules in one process (alternating, same clocks regime)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from probe_perf import make_store, make_queries, timeit
from paper_2506_21593_b200 import MODE_TENSOR
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
idx = make_store(n, 1024)
q = make_queries(idx, 4096, 1024)
import ctypes
res = {"persistent": [], "waves": []}
for rep in range(6):
    for name in ("persistent", "waves"):
        os.environ["PR_TC_SCHEDULE"] = name
        # the library reads the env var once per process: use a fresh ctypes getenv-less flag via setenv
        ctypes.CDLL(None).setenv(b"PR_TC_SCHEDULE", name.encode(), 1)
        res[name].append(timeit(lambda: idx.search_batch(q, 5, mode=MODE_TENSOR, validate=False), reps=3))
for k, v in res.items():
    print(k, ["%.2f" % x for x in v], "min %.2f" % min(v))
