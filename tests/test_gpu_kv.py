"""GPU fixed-KV table vs a dict oracle (reference caches.py:45-101)."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _arena(texts):
    import torch

    bs = [t.encode("utf-8", "surrogatepass") for t in texts]
    off = np.zeros(len(bs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(b) for b in bs])
    data = np.frombuffer(b"".join(bs) or b"\0", dtype=np.uint8).copy()
    return torch.from_numpy(data).cuda(), torch.from_numpy(off).cuda()


def test_fingerprint_host_equals_device(gpu):
    import torch

    from paper_2506_21593_b200 import _lib

    L = _lib.load()
    texts = ["", "a", "Q1", "q1", "Who wrote Hamlet?", "Who wrote Hamlet? ", "x" * 15, "y" * 16, "z" * 17,
             "ünïcödé ✓", "query-000000001"]
    data, off = _arena(texts)
    fp = torch.empty((len(texts), 2), dtype=torch.int64, device="cuda")
    _lib.check(L.pr_fingerprint(_lib.ptr(data), _lib.ptr(off), len(texts), _lib.ptr(fp), _lib.stream_ptr()))
    dev = fp.cpu().numpy().view(np.uint64)
    for i, t in enumerate(texts):
        b = t.encode("utf-8")
        out = (ctypes.c_uint64 * 2)()
        buf = ctypes.create_string_buffer(b, len(b))
        L.pr_fingerprint_host(ctypes.cast(buf, ctypes.c_void_p), len(b), out)
        assert (out[0], out[1]) == (int(dev[i, 0]), int(dev[i, 1])), t
    assert len({(int(a), int(b)) for a, b in dev}) == len(texts)


def test_put_get_last_write_wins_and_erase(gpu):
    import torch

    from paper_2506_21593_b200 import _lib

    L = _lib.load()
    h = ctypes.c_void_p()
    _lib.check(L.pr_kv_create(16, ctypes.byref(h)))
    rng = np.random.default_rng(3)
    keys = [f"query-{i:09d}" for i in range(5000)]
    oracle: dict[str, int] = {}
    seq = 0
    for batch in range(6):
        pick = rng.integers(0, len(keys), size=3000)  # duplicates inside a batch
        texts = [keys[i] for i in pick]
        vals = np.arange(seq, seq + len(texts), dtype=np.int64)
        seq += len(texts)
        for t, v in zip(texts, vals):
            oracle[t] = int(v)
        data, off = _arena(texts)
        fp = torch.empty((len(texts), 2), dtype=torch.int64, device="cuda")
        _lib.check(L.pr_fingerprint(_lib.ptr(data), _lib.ptr(off), len(texts), _lib.ptr(fp), _lib.stream_ptr()))
        v = torch.from_numpy(vals).cuda()
        _lib.check(L.pr_kv_put(h, _lib.ptr(fp), _lib.ptr(v), len(texts), _lib.stream_ptr()))
    probe = keys + ["absent-" + k for k in keys[:1000]] + ["query-00000001", "Query-000000001"]
    data, off = _arena(probe)
    out = torch.empty(len(probe), dtype=torch.int64, device="cuda")
    hit = torch.empty(len(probe), dtype=torch.uint8, device="cuda")
    _lib.check(L.pr_kv_get_text(h, _lib.ptr(data), _lib.ptr(off), len(probe), _lib.ptr(out), _lib.ptr(hit),
                                _lib.stream_ptr()))
    out, hit = out.cpu().numpy(), hit.cpu().numpy()
    for i, t in enumerate(probe):
        if t in oracle:
            assert hit[i] == 1 and out[i] == oracle[t], t
        else:
            assert hit[i] == 0 and out[i] == -1, t
    assert L.pr_kv_size(h) == len(oracle)
    # erase half, re-probe
    gone = list(oracle)[::2]
    data, off = _arena(gone)
    fp = torch.empty((len(gone), 2), dtype=torch.int64, device="cuda")
    _lib.check(L.pr_fingerprint(_lib.ptr(data), _lib.ptr(off), len(gone), _lib.ptr(fp), _lib.stream_ptr()))
    _lib.check(L.pr_kv_erase(h, _lib.ptr(fp), len(gone), _lib.stream_ptr()))
    assert L.pr_kv_size(h) == len(oracle) - len(gone)
    data, off = _arena(list(oracle))
    out = torch.empty(len(oracle), dtype=torch.int64, device="cuda")
    hit = torch.empty(len(oracle), dtype=torch.uint8, device="cuda")
    _lib.check(L.pr_kv_get_text(h, _lib.ptr(data), _lib.ptr(off), len(oracle), _lib.ptr(out), _lib.ptr(hit),
                                _lib.stream_ptr()))
    hit = hit.cpu().numpy()
    gs = set(gone)
    for i, t in enumerate(oracle):
        assert hit[i] == (0 if t in gs else 1)
    L.pr_kv_destroy(h)


def test_sharded_kv_single_rank_device_path(gpu):
    from paper_2506_21593_b200.sharded_kv import ShardedKV

    kv = ShardedKV(capacity=10000)
    keys = [f"query-{i:09d}" for i in range(5000)]
    kv.put(keys + keys[:7], list(range(5000)) + [9000 + i for i in range(7)])
    vals, hit = kv.get(keys + ["absent", "query-00000000"])
    vals = vals.cpu().numpy()
    assert list(vals[:7]) == [9000 + i for i in range(7)]
    assert list(vals[7:5000]) == list(range(7, 5000))
    assert vals[5000] == -1 and vals[5001] == -1 and not bool(hit[5000])
