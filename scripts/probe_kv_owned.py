"""Per-rank cost of the hash-partitioned fixed-KV lookup (sharded_kv.py): rank 0's
pr_kv_get_text_owned over a batch of B keys, for world = 1, 2, 4, 8, with rank 0's table
holding only the keys it owns (100M / world).  The kernel hashes every key once and probes
only the owned ones, so its time should fall towards the hashing floor as world grows.
(One GPU: each world size is timed as rank 0 alone.)"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from benchlib.configs import _key_arena  # noqa: E402
from paper_2506_21593_b200 import _lib  # noqa: E402

L = _lib.load()
s = _lib.stream_ptr()
n_keys = int(os.environ.get("KV_KEYS", 100_000_000))
B, reps = 1 << 22, 20
rng = np.random.default_rng(5)
ids = np.concatenate([rng.integers(0, n_keys, B // 2), rng.integers(n_keys, 2 * n_keys, B - B // 2)])
rng.shuffle(ids)
qbuf, qoff = _key_arena(ids)
d_qb, d_qo = torch.from_numpy(qbuf).cuda(), torch.from_numpy(qoff).cuda()
out = torch.empty(B, dtype=torch.int64, device="cuda")
hit = torch.empty(B, dtype=torch.uint8, device="cuda")
res = {}
for world in (1, 2, 4, 8):
    h = ctypes.c_void_p()
    _lib.check(L.pr_kv_create(n_keys // world + 1, ctypes.byref(h)))
    for c0 in range(0, n_keys, 8_000_000):
        kid = np.arange(c0, min(n_keys, c0 + 8_000_000), dtype=np.int64)
        buf, off = _key_arena(kid)
        d_b, d_o, v = torch.from_numpy(buf).cuda(), torch.from_numpy(off).cuda(), torch.from_numpy(kid).cuda()
        _lib.check(L.pr_kv_put_text_owned(h, _lib.ptr(d_b), _lib.ptr(d_o), kid.size, int(off[-1]), _lib.ptr(v), 0, world, s))
    torch.cuda.synchronize()
    for _ in range(3):
        _lib.check(L.pr_kv_get_text_owned(h, _lib.ptr(d_qb), _lib.ptr(d_qo), B, 0, world, _lib.ptr(out), _lib.ptr(hit), s))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        _lib.check(L.pr_kv_get_text_owned(h, _lib.ptr(d_qb), _lib.ptr(d_qo), B, 0, world, _lib.ptr(out), _lib.ptr(hit), s))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    size = int(L.pr_kv_size(h, s))
    res[world] = {"rank0_keys": size, "ms_per_4M_batch": round(ms, 4), "G_keys_per_s": round(B / ms / 1e6, 2)}
    L.pr_kv_destroy(h)
print(json.dumps({"batch": B, "table_keys_total": n_keys, "per_world": res}))
