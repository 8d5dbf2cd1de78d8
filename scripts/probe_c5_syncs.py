"""Where does the C5 host path block on the device?  Replays sessions with torch's sync
debug mode on and tallies the Python call sites of every synchronising torch op
(measurement only; C-level syncs inside libpentarag do not show here)."""
from __future__ import annotations

import collections
import os
import sys
import traceback
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from benchlib import configs as C  # noqa: E402

sites = collections.Counter()


def show(message, category, filename, lineno, file=None, line=None):
    st = [f for f in traceback.extract_stack()[:-1] if "paper_2506_21593_b200" in f.filename or "benchlib" in f.filename]
    key = " <- ".join(f"{os.path.basename(f.filename)}:{f.lineno}:{f.name}" for f in st[-3:][::-1])
    sites[key] += 1


n = int(os.environ.get("C5_ROWS", 2_000_000))
idx = bench.build_shard(n, 1024, 0, n)
torch.cuda.synchronize()
orig = C.c5_routed


warnings.showwarning = show
warnings.simplefilter("always")
_real_sync = C._events


def events_hook():
    torch.cuda.set_sync_debug_mode("warn")
    return _real_sync()


C._events = events_hook
r = C.c5_routed(idx, n, n_sessions=2, queries_per_session=8192, parity_queries=0, l5_oracle_queries=0)
torch.cuda.set_sync_debug_mode("default")
print("value", r["value"])
for k, v in sites.most_common(40):
    print(f"{v:6d}  {k}")
