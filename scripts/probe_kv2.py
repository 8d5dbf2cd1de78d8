"""KV probe kernel under a profiler: 100M-key table, then pr_kv_get_text launches at
B=65536 (x4) and one 4M-key batch.  Used with ncu (-k regex:kv_get) for the C3 kernel."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from benchlib.configs import _key_arena  # noqa: E402
from paper_2506_21593_b200 import _lib  # noqa: E402

n_keys = int(os.environ.get("KV_KEYS", 100_000_000))
L = _lib.load()
if os.environ.get("PR_L2FETCH"):
    _lib.check(L.pr_l2_fetch_granularity(int(os.environ["PR_L2FETCH"]), None))
h = ctypes.c_void_p()
_lib.check(L.pr_kv_create(n_keys, ctypes.byref(h)))
s = _lib.stream_ptr()
for c0 in range(0, n_keys, 8_000_000):
    ids = np.arange(c0, min(n_keys, c0 + 8_000_000), dtype=np.int64)
    buf, off = _key_arena(ids)
    d_buf, d_off = torch.from_numpy(buf).cuda(), torch.from_numpy(off).cuda()
    vals = torch.from_numpy(ids).cuda()
    _lib.check(L.pr_kv_put_text(h, _lib.ptr(d_buf), _lib.ptr(d_off), ids.size, int(off[-1]), _lib.ptr(vals), s))
torch.cuda.synchronize()
rng = np.random.default_rng(3)
for B in [65536] * 4 + [4 << 20]:
    ids = np.concatenate([rng.integers(0, n_keys, B // 2), rng.integers(n_keys, 2 * n_keys, B - B // 2)])
    rng.shuffle(ids)
    buf, off = _key_arena(ids)
    d_buf, d_off = torch.from_numpy(buf).cuda(), torch.from_numpy(off).cuda()
    out = torch.empty(B, dtype=torch.int64, device="cuda")
    hit = torch.empty(B, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(L.pr_kv_get_text(h, _lib.ptr(d_buf), _lib.ptr(d_off), B, _lib.ptr(out), _lib.ptr(hit), s))
    torch.cuda.synchronize()
    want = torch.from_numpy(np.where(ids < n_keys, ids, -1)).cuda()
    print(B, "mismatches", int((out != want).sum().item()), f"{(time.perf_counter() - t0) * 1e6:.1f} us wall")
