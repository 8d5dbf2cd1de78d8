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


def _table(L, cap=16, flags=0):
    from paper_2506_21593_b200 import _lib

    h = ctypes.c_void_p()
    _lib.check(L.pr_kv_create_ex(cap, flags, ctypes.byref(h)))
    return h


def _put(L, h, texts, vals):
    import torch

    from paper_2506_21593_b200 import _lib

    data, off = _arena(texts)
    nbytes = int(off[-1].item())
    v = torch.as_tensor(np.asarray(vals, dtype=np.int64)).cuda()
    _lib.check(L.pr_kv_put_text(h, _lib.ptr(data), _lib.ptr(off), len(texts), nbytes, _lib.ptr(v),
                                _lib.stream_ptr()))


def _get(L, h, texts):
    import torch

    from paper_2506_21593_b200 import _lib

    data, off = _arena(texts)
    out = torch.empty(len(texts), dtype=torch.int64, device="cuda")
    hit = torch.empty(len(texts), dtype=torch.uint8, device="cuda")
    _lib.check(L.pr_kv_get_text(h, _lib.ptr(data), _lib.ptr(off), len(texts), _lib.ptr(out), _lib.ptr(hit),
                                _lib.stream_ptr()))
    return out.cpu().numpy(), hit.cpu().numpy()


def _erase(L, h, texts):
    from paper_2506_21593_b200 import _lib

    data, off = _arena(texts)
    _lib.check(L.pr_kv_erase_text(h, _lib.ptr(data), _lib.ptr(off), len(texts), _lib.stream_ptr()))


def _check(L, h, oracle, probe):
    from paper_2506_21593_b200 import _lib

    out, hit = _get(L, h, probe)
    for i, t in enumerate(probe):
        if t in oracle:
            assert hit[i] == 1 and out[i] == oracle[t], t
        else:
            assert hit[i] == 0 and out[i] == -1, t
    assert L.pr_kv_size(h, _lib.stream_ptr()) == len(oracle)


@pytest.mark.parametrize("flags", [0, 1])
def test_put_get_last_write_wins_and_erase(gpu, flags):
    """Dict oracle (caches.py:57-77) over batched upserts with in-batch duplicates, table
    growth from 16 slots, erase and re-insert.  flags=1 (PR_KV_WEAK_HASH) keeps 2 tag bits
    and 4 home buckets, so distinct keys collide on tag and bucket all the time: every
    answer must still be byte-exact (a clash is a miss, never another key's value)."""
    from paper_2506_21593_b200 import _lib

    L = _lib.load()
    h = _table(L, 16, flags)
    rng = np.random.default_rng(3)
    nkeys = 5000 if flags == 0 else 600
    keys = [f"query-{i:09d}" for i in range(nkeys)]
    keys += ["Who wrote Hamlet?", "Who wrote Hamlet? ", "who wrote Hamlet?", "ünïcödé ✓", "x" * 40, "x" * 41,
             "", "a"]
    oracle: dict[str, int] = {}
    seq = 0
    for batch in range(6):
        pick = rng.integers(0, len(keys), size=min(3000, 2 * len(keys)))  # duplicates inside a batch
        texts = [keys[i] for i in pick]
        vals = np.arange(seq, seq + len(texts), dtype=np.int64)
        seq += len(texts)
        for t, v in zip(texts, vals):
            oracle[t] = int(v)
        _put(L, h, texts, vals)
    probe = keys + ["absent-" + k for k in keys[:500]] + ["query-00000001", "Query-000000001", "x" * 39]
    _check(L, h, oracle, probe)
    gone = list(oracle)[::2]
    _erase(L, h, gone)
    for t in gone:
        del oracle[t]
    _check(L, h, oracle, probe)
    # re-insert some erased keys (tombstones are skipped, new records appended)
    back = gone[::3]
    _put(L, h, back, np.arange(seq, seq + len(back)))
    for i, t in enumerate(back):
        oracle[t] = seq + i
    _check(L, h, oracle, probe)
    L.pr_kv_destroy(h)


def test_fingerprint_clash_is_a_miss(gpu):
    """Forced clash: under PR_KV_WEAK_HASH many keys share tag AND home bucket; probing a
    key that is absent but shares its tag with stored keys must miss, and each stored key
    must return its own value (the reference dict compares bytes, caches.py:57-65)."""
    from paper_2506_21593_b200 import _lib

    L = _lib.load()
    h = _table(L, 64, 1)
    stored = [f"k{i}" for i in range(40)]
    _put(L, h, stored, np.arange(40) * 10)
    out, hit = _get(L, h, stored + [f"k{i}" for i in range(40, 400)])
    assert list(out[:40]) == list(np.arange(40) * 10) and hit[:40].all()
    assert (out[40:] == -1).all() and not hit[40:].any()
    L.pr_kv_destroy(h)


def test_kv_arena_compaction_bounds_memory(gpu):
    """FixedKVCache host arena follows the live keys: overwriting the same
    keys many times keeps it bounded, and export order stays write order."""
    from paper_2506_21593_b200 import AnswerRecord, FixedKVCache, LayerTag

    kv = FixedKVCache()
    keys = [f"q{i}" for i in range(300)]
    for r in range(60):
        kv.put_many(keys, [AnswerRecord(text=f"{k}-{r}", layer=LayerTag.FIXED_KV, confidence=0.9) for k in keys])
    assert len(kv) == 300
    assert len(kv._arena) <= 2 * kv._COMPACT_MIN
    assert kv.get("q7").text == "q7-59"
    ex = kv.export_entries()
    assert [e["query_text"] for e in ex] == keys and ex[0]["answer"]["text"] == "q0-59"


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


def test_owned_probe_matches_host_owner(gpu):
    """pr_kv_get_text_owned / pr_kv_put_text_owned act exactly on the keys owner_host gives
    the rank; the union over ranks is the unsharded table."""
    import torch

    from paper_2506_21593_b200 import _lib
    from paper_2506_21593_b200.sharded_kv import owner_host

    L = _lib.load()
    world = 4
    keys = [f"query-{i:09d}" for i in range(3000)]
    data, off = _arena(keys)
    vals = torch.arange(len(keys), dtype=torch.int64, device="cuda")
    got = np.full(len(keys), -1)
    for r in range(world):
        h = _table(L, 4096)
        _lib.check(L.pr_kv_put_text_owned(h, _lib.ptr(data), _lib.ptr(off), len(keys), int(off[-1].item()),
                                          _lib.ptr(vals), r, world, _lib.stream_ptr()))
        assert L.pr_kv_size(h, _lib.stream_ptr()) == sum(owner_host(k, world) == r for k in keys)
        out = torch.empty(len(keys), dtype=torch.int64, device="cuda")
        hit = torch.empty(len(keys), dtype=torch.uint8, device="cuda")
        _lib.check(L.pr_kv_get_text_owned(h, _lib.ptr(data), _lib.ptr(off), len(keys), r, world, _lib.ptr(out),
                                          _lib.ptr(hit), _lib.stream_ptr()))
        o = out.cpu().numpy()
        mine = np.array([owner_host(k, world) == r for k in keys])
        assert (o[~mine] == -1).all() and (o[mine] >= 0).all()
        got = np.maximum(got, o)
        L.pr_kv_destroy(h)
    assert (got == np.arange(len(keys))).all()
