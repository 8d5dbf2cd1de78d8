"""C3 alone (benchlib.configs.c3_kv); PR_L2FETCH=<bytes> sets the L2 fetch granularity first."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from benchlib import configs as C  # noqa: E402
from paper_2506_21593_b200 import _lib  # noqa: E402

prev = ctypes.c_int()
_lib.check(_lib.load().pr_l2_fetch_granularity(int(os.environ.get("PR_L2FETCH", "0")), ctypes.byref(prev)))
now = ctypes.c_int()
_lib.check(_lib.load().pr_l2_fetch_granularity(0, ctypes.byref(now)))
r = C.c3_kv(6539.2, streams=int(os.environ.get("C3_STREAMS", "8")))
r["l2_fetch_granularity"] = {"before": prev.value, "used": now.value}
print(json.dumps(r))
