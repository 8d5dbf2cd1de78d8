"""Quick perf probe of the search paths (not the bench; prints one line per case)."""
from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2506_21593_b200 import MODE_EXACT, MODE_TENSOR, MODE_TENSOR_I8, FlatIndex  # noqa: E402


def make_store(n, d, seed=7, chunk=1 << 20):
    idx = FlatIndex(dim=d, capacity=n)
    g = torch.Generator(device="cuda").manual_seed(seed)
    for r0 in range(0, n, chunk):
        m = min(chunk, n - r0)
        x = torch.randn((m, d), generator=g, device="cuda", dtype=torch.float32)
        x = (x.double() / x.double().norm(dim=1, keepdim=True)).float()
        idx.extend_arrays([str(r0 + i) for i in range(m)], x, validate=False)
        del x
    return idx


def make_queries(idx, b, d, frac_dup=0.25, seed=11):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn((b, d), generator=g, device="cuda")
    ndup = int(b * frac_dup)
    rows = torch.randint(0, len(idx), (ndup,), generator=g, device="cuda")
    base = torch.stack([idx.read_rows(int(r), 1)[0] for r in rows.tolist()]) if ndup else None
    if ndup:
        q[:ndup] = base + 0.3 * q[:ndup] / q[:ndup].norm(dim=1, keepdim=True)
    q = (q.double() / q.double().norm(dim=1, keepdim=True)).float()
    return q.contiguous()


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="1000000x1024x4096x5,1000000x768x4096x1,10000000x1024x4096x5")
    ap.add_argument("--exact", action="store_true")
    a = ap.parse_args()
    for case in a.cases.split(","):
        n, d, b, k = (int(x) for x in case.split("x"))
        t0 = time.time()
        idx = make_store(n, d)
        q = make_queries(idx, b, d)
        torch.cuda.synchronize()
        build_s = time.time() - t0
        flop = 2.0 * n * d * b
        ref = None
        for name, mode in (("TC16", MODE_TENSOR), ("TC8", MODE_TENSOR_I8)):
            idx.set_timing(True)
            ms = timeit(lambda: idx.search_batch(q, k, mode=mode, validate=False))
            kms, kn = idx.scan_time()
            st = idx.stats()
            res = idx.search_batch(q, k, mode=mode, validate=False)
            rows = res.rows.cpu()
            same = "" if ref is None else f" rows==TC16: {bool((rows == ref).all())}"
            ref = rows if ref is None else ref
            print(f"{name} n={n} d={d} B={b} k={k}: {ms:.2f} ms  {b / ms * 1e3:.0f} q/s  "
                  f"{flop / ms / 1e9:.1f} TOP/s(e2e)  scan {kms / max(kn, 1):.2f} ms/launch "
                  f"nsplit={st.nsplit} fallback={st.fallback} cand={st.candidates} appended={st.appended} "
                  f"build={build_s:.1f}s{same}", flush=True)
        if a.exact:
            bq = min(b, 256)
            ms = timeit(lambda: idx.search_batch(q[:bq], k, mode=MODE_EXACT, validate=False), reps=1)
            print(f"EX  n={n} d={d} B={bq} k={k}: {ms:.2f} ms  {bq / ms * 1e3:.1f} q/s "
                  f"{n * d * bq / ms / 1e9:.2f} TFMA/s", flush=True)
        del idx, q
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
