"""C2 (semantic cache 1M x 768, batch 4096, top-1 + threshold) alone."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from benchlib import configs as C  # noqa: E402

r = C.c2_semantic(2760.0, "probe", None, steps=int(os.environ.get("STEPS", "20")))
print("c2", round(r["value"] / 1e6, 3), "M/s", round(r["ms_per_batch"], 3), "ms/batch kernel", round(r["roofline"]["kernel_ms"], 3),
      "ms parity", r["parity"])
