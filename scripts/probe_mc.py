"""Int8 scan: CTA pairs per multicast cluster (PR_I8_MC = 1 / 2 / 4) at the C4 shape.

Continuous blocks of searches per setting (the scan is power-capped: alternating single
calls share one power-averaging window), repeated round-robin; per block: mean ms per
search, in-library scan-kernel ms, median SM clock sampled during the block, and the
result rows compared with the first setting's.
"""
from __future__ import annotations

import argparse
import os
import statistics
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from scripts.probe_perf import make_queries, make_store  # noqa: E402
from paper_2506_21593_b200 import MODE_TENSOR_I8  # noqa: E402


class Clocks:
    def __init__(self):
        self.samples = []
        self.p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                                   "-lms", "100", "-i", "0"], stdout=subprocess.PIPE, text=True)
        threading.Thread(target=self._rd, daemon=True).start()

    def _rd(self):
        for ln in self.p.stdout:
            try:
                c, w = (float(x) for x in ln.split(","))
                self.samples.append((time.time(), c, w))
            except ValueError:
                pass

    def window(self, t0, t1):
        s = [(c, w) for t, c, w in self.samples if t0 <= t <= t1]
        if not s:
            return None, None
        return statistics.median(c for c, _ in s), statistics.median(w for _, w in s)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="10000000x1024x4096x5")
    ap.add_argument("--mcs", default="1,2,4", help="settings MC[:NSPLIT[:ENV=VAL...]] (NSPLIT 0 = auto)")
    ap.add_argument("--block", type=int, default=40)
    ap.add_argument("--rounds", type=int, default=3)
    a = ap.parse_args()
    n, d, b, k = (int(x) for x in a.case.split("x"))
    idx = make_store(n, d)
    q = make_queries(idx, b, d)
    torch.cuda.synchronize()
    clk = Clocks()
    ref = None
    res = {}
    for r in range(a.rounds):
        for mc in a.mcs.split(","):
            parts = mc.split(":")
            os.environ["PR_I8_MC"] = parts[0]
            os.environ["PR_I8_NSPLIT"] = parts[1] if len(parts) > 1 else "0"
            for kv in parts[2:]:
                key, val = kv.split("=")
                os.environ[key] = val
            out = idx.search_batch(q, k, mode=MODE_TENSOR_I8, validate=False)
            rows = out.rows.cpu()
            same = True if ref is None else bool((rows == ref).all())
            ref = rows if ref is None else ref
            idx.set_timing(True)
            idx.scan_time()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.time()
            s.record()
            for _ in range(a.block):
                idx.search_batch(q, k, mode=MODE_TENSOR_I8, validate=False)
            e.record()
            torch.cuda.synchronize()
            t1 = time.time()
            kms, kn = idx.scan_time()
            ms = s.elapsed_time(e) / a.block
            c, w = clk.window(t0 + 0.3 * (t1 - t0), t1)
            st = idx.stats()
            res.setdefault(mc, []).append(ms)
            for kv in parts[2:]:
                os.environ.pop(kv.split("=")[0], None)
            print(f"round {r} MC={mc}: {ms:.2f} ms/search ({b / ms * 1e3:.0f} q/s) scan {kms / max(kn, 1):.2f} ms "
                  f"nsplit={st.nsplit} clock {c} MHz power {w} W rows==MC{a.mcs.split(',')[0]}: {same}", flush=True)
    for mc, v in res.items():
        print(f"MC={mc}: median {statistics.median(v):.2f} ms/search over {len(v)} blocks")
    clk.p.terminate()


if __name__ == "__main__":
    main()
