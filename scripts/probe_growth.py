"""Find slow store-maintenance calls in the C5 replay: every FlatIndex append /
search is bracketed by device syncs and reported when it takes > 10 ms."""
from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from benchlib import configs as C  # noqa: E402
from paper_2506_21593_b200 import index as I  # noqa: E402
from scripts.probe_perf import make_store  # noqa: E402


def wrap(name, cls=I.FlatIndex, thr=10.0):
    orig = getattr(cls, name)

    def f(self, *a, **kw):
        torch.cuda.synchronize()
        n0 = len(self) if hasattr(self, "__len__") else 0
        t = time.perf_counter()
        c = time.thread_time()
        r = orig(self, *a, **kw)
        cpu_in = (time.thread_time() - c) * 1e3
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
        if ms > thr:
            free, tot = torch.cuda.mem_get_info()
            extra = ""
            if name == "search_batch":
                st = self.stats()
                extra = (f" nq={a[0].shape[0]} k={a[1]} limit={kw.get('row_limit') is not None} path={st.path} "
                         f"fallback={st.fallback} collected={st.collected} cand={st.candidates} "
                         f"appended={st.appended} nsplit={st.nsplit}")
            print(f"{name}: {ms:.1f} ms (thread cpu {cpu_in:.1f} ms before sync) rows {n0}->{len(self)} free {free / 2**30:.1f} GiB{extra}", flush=True)
        return r

    setattr(cls, name, f)


for nm in ("extend_arrays", "append_rows_from", "append_anonymous_from", "truncate", "clear"):
    wrap(nm, thr=3.0)
wrap("search_batch")
from paper_2506_21593_b200 import knowledge as K  # noqa: E402
wrap("settle_from_rows", K.AdaptiveKnowledgeMemory, 3.0)
n = int(os.environ.get("N", "10000000"))
store = make_store(n, 1024)
print("store built; free GiB", torch.cuda.mem_get_info()[0] / 2**30, "torch reserved GiB",
      torch.cuda.memory_reserved() / 2**30, flush=True)
import gc  # noqa: E402

_gc_t = {}


def _gc_cb(phase, info):
    if phase == "start":
        _gc_t["t"] = time.perf_counter()
    else:
        ms = (time.perf_counter() - _gc_t["t"]) * 1e3
        if ms > 3:
            print(f"gc gen{info['generation']}: {ms:.1f} ms collected {info['collected']}", flush=True)


gc.callbacks.append(_gc_cb)
if os.environ.get("FREEZE"):
    gc.collect()
    gc.freeze()
    print("frozen", gc.get_freeze_count(), flush=True)
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)), "loadavg", os.getloadavg(), flush=True)
r = C.c5_routed(store, n, n_sessions=2, queries_per_session=20000, parity_queries=0)
print("value", r["value"])
