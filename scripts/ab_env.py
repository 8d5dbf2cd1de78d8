"""Interleaved A/B of a search-path environment knob inside ONE process (the
library reads PR_* knobs per call), so clock/power drift hits both arms alike.

    python scripts/ab_env.py --case 10000000x1024x4096x5 --var PR_I8_REFINE --a 1 --b 0 --reps 12
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2506_21593_b200 import MODE_TENSOR_I8  # noqa: E402
from scripts.probe_perf import make_queries, make_store  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="10000000x1024x4096x5")
    ap.add_argument("--var", required=True)
    ap.add_argument("--a", required=True)
    ap.add_argument("--b", required=True)
    ap.add_argument("--reps", type=int, default=12)
    ap.add_argument("--mode", type=int, default=MODE_TENSOR_I8)
    a = ap.parse_args()
    n, d, b, k = (int(x) for x in a.case.split("x"))
    idx = make_store(n, d)
    q = make_queries(idx, b, d)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = {a.a: [], a.b: []}
    ref = None
    for r in range(a.reps + 1):
        for val in (a.a, a.b) if r % 2 == 0 else (a.b, a.a):
            os.environ[a.var] = val
            torch.cuda.synchronize()
            s.record()
            res = idx.search_batch(q, k, mode=a.mode, validate=False)
            e.record()
            torch.cuda.synchronize()
            if r > 0:
                times[val].append(s.elapsed_time(e))
            rows = res.rows.cpu()
            ref = rows if ref is None else ref
            assert bool((rows == ref).all()), f"{a.var}={val}: results differ"
    for val in (a.a, a.b):
        t = times[val]
        print(f"{a.var}={val}: median {statistics.median(t):.2f} ms  min {min(t):.2f}  max {max(t):.2f}  "
              f"({b / statistics.median(t) * 1e3:.0f} q/s)", flush=True)
    st = idx.stats()
    print(f"appended(last)={st.appended} rescored(last)={st.candidates}")


if __name__ == "__main__":
    main()
