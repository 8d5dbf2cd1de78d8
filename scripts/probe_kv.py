"""C3 (fixed KV, 100M keys) alone: graph-replayed 65536-key batches and the 4M-key batch."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from benchlib import configs as C  # noqa: E402

r = C.c3_kv(6539.2, n_keys=int(os.environ.get("KEYS", "100000000")))
print(os.environ.get("PR_LIB", "in-tree"), "graph", round(r["value"] / 1e9, 3), "G/s", round(r["us_per_batch"], 2), "us/batch",
      "eager", round(r["eager"]["value"] / 1e9, 3), "large", round(r["large_batch"]["value"] / 1e9, 3), "G/s",
      "parity", r["parity"])
