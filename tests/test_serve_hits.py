"""CPU test of the cascade's vectorised cache-hit pass (cascade._serve_hits) against the
per-query replay it replaces: a hit serves the latest answer written for its key by an
earlier query of the span, else by the previous span, else the stored entry
(reference semantics: router.py:333-337 writes every routed query back before the next)."""
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2506_21593_b200 import cascade
from paper_2506_21593_b200.caches import CacheEntry
from paper_2506_21593_b200.ledger import BatchLedger, entries_of, entry_text_conf


def _ledger(texts, answers, conf):
    lg = BatchLedger.__new__(BatchLedger)
    lg.text, lg.conf = list(answers), np.asarray(conf, dtype=np.float64)
    return lg, entries_of(texts, lg, 0)


def _replay(sp, hit_js, is_l1, sc_row, kv_val, text, conf_l, sc_ids, kv_arena, sc_payloads):
    """The straightforward per-hit loop (the pre-vectorisation code)."""
    texts = sp.texts
    latest, nxt = {}, 0
    for j in hit_js.tolist():
        latest.update(zip(texts[nxt:j], range(nxt, j)))
        nxt = j
        key = texts[j] if is_l1[j] else sc_ids[int(sc_row[j])]
        i = latest.get(key, -1)
        if i >= 0:
            text[j], conf_l[j] = text[i], conf_l[i]
        elif sp.prev_last is not None and key in sp.prev_last:
            text[j], conf_l[j] = entry_text_conf(sp.prev.entries[sp.prev_last[key]])
        elif is_l1[j]:
            text[j], conf_l[j] = entry_text_conf(kv_arena[int(kv_val[j])])
        else:
            text[j], conf_l[j] = entry_text_conf(sc_payloads[int(sc_row[j])])


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("mixed_entries", [False, True])
def test_serve_hits_equals_replay(seed, mixed_entries):
    rng = np.random.default_rng(seed)
    vocab = [f"q{i}" for i in range(int(rng.integers(5, 60)))]
    B = int(rng.integers(1, 300))
    texts = [vocab[i] for i in rng.integers(0, len(vocab), B)]
    # stores: every vocabulary text has a stored KV entry and semantic-cache row
    old_lg, old_entries = _ledger(vocab, [f"old-{t}" for t in vocab], rng.random(len(vocab)))
    kv_arena = list(old_entries)
    if mixed_entries:  # entries written by route() (CacheEntry) beside batch-written ones
        kv_arena[0] = CacheEntry(vocab[0], SimpleNamespace(text="ce-answer", confidence=0.25), 0)
    sc_ids = list(vocab)
    sc_payloads = list(kv_arena)
    prev = None
    prev_last = None
    if rng.random() < 0.7:
        pt = [vocab[i] for i in rng.integers(0, len(vocab), int(rng.integers(1, 80)))]
        _, pentries = _ledger(pt, [f"prev-{t}-{j}" for j, t in enumerate(pt)], rng.random(len(pt)))
        prev = SimpleNamespace(entries=pentries, texts=pt, B=len(pt))
        prev_last = dict(zip(pt, range(len(pt))))
    first_of = dict(zip(reversed(texts), range(B - 1, -1, -1)))
    first = np.fromiter(map(first_of.__getitem__, texts), dtype=np.int64, count=B)
    sp = SimpleNamespace(texts=texts, first=first, first_of=first_of, prev=prev, prev_last=prev_last)
    serving = rng.integers(0, 3, B)  # 0: answered by retrieval, 1: L1 hit, 2: L2 hit
    is_l1 = serving == 1
    hit_js = np.flatnonzero(serving > 0)
    kv_val = np.array([vocab.index(t) for t in texts], dtype=np.int64)
    sc_row = rng.integers(0, len(vocab), B).astype(np.int64)
    base_text = [None if serving[j] else f"retr-{j}" for j in range(B)]
    base_conf = [0.0 if serving[j] else float(rng.random()) for j in range(B)]
    router = SimpleNamespace(kv_cache=SimpleNamespace(entry_at=kv_arena.__getitem__),
                             semantic_cache=SimpleNamespace(index=SimpleNamespace(
                                 _ids=sc_ids, payload_at=sc_payloads.__getitem__)))
    want_t, want_c = list(base_text), list(base_conf)
    _replay(sp, hit_js, is_l1, sc_row, kv_val, want_t, want_c, sc_ids, kv_arena, sc_payloads)
    got_t, got_c = list(base_text), list(base_conf)
    if hit_js.size:
        cascade._serve_hits(router, sp, hit_js, is_l1, sc_row, kv_val, got_t, got_c)
    assert got_t == want_t
    assert np.array_equal(np.asarray(got_c, dtype=np.float64), np.asarray(want_c, dtype=np.float64))
