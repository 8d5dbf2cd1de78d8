"""One C4-shaped int8 search per setting with PR_I8_VERBOSE: split/cluster choice,
cooperative-path rate, flagged groups, appended and rescored rows (measurement only)."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from scripts.probe_perf import make_queries, make_store  # noqa: E402
from paper_2506_21593_b200 import MODE_TENSOR_I8  # noqa: E402

n, d, b, k = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "10000000x1024x4096x5").split("x"))
idx = make_store(n, d)
q = make_queries(idx, b, d)
os.environ["PR_I8_VERBOSE"] = "1"
for setting in (sys.argv[2] if len(sys.argv) > 2 else "PR_I8_PILOT_STRIDE=32").split(","):
    key, val = setting.split("=")
    os.environ[key] = val
    for half in ("all", "planted", "random"):
        qq = q if half == "all" else (q[: b // 4] if half == "planted" else q[b // 4:])
        idx.search_batch(qq, k, mode=MODE_TENSOR_I8, validate=False)
        torch.cuda.synchronize()
        st = idx.stats()
        print(f"{setting} {half}: appended={st.appended} ({st.appended / len(qq):.1f}/query) "
              f"rescored={st.candidates} fallback={st.fallback}", file=sys.stderr, flush=True)
    os.environ.pop(key)
