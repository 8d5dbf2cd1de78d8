"""Generate golden fixtures by running the REAL reference (ragcascade) here.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Only this script reads /root/reference; the fixtures it writes are small,
committed, and are what the tests (CPU and GPU) compare against — the GPU
box never sees the reference.

Fixtures:
  flat_index.npz   FlatIndex.search (index.py:155-189) on seeded stores with
                   injected duplicate ties, tie-heavy and self-snap probes,
                   one-hot / orthogonal cases: entry rows, exact fp64 scores
  embed.json       HashEmbedder (embedding.py:117-160) vectors for fixed texts
  kv_ops.json      FixedKVCache get/put/LRU op sequence and results
  router_trace.json  CascadeRouter.route (router.py:275-364) over a seeded
                   replay (simulation.next_query) on a 60-row KB: per-query
                   probes, serving layer, answer text, supporting passages,
                   and the final store counters
  simulation.json  run_simulation(2 sessions x 150 queries) session logs
  snapshot.json    FlatIndex.snapshot bytes (RCFLATIX, index.py:198-220) of an index
                   with upserts + payloads, restore() results (index.py:222-261) for
                   it and for crafted duplicate-id / invalid-vector / corrupt blobs

    python tests/golden/make_golden.py snapshot   # regenerate snapshot.json only
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import ragcascade as rc  # noqa: E402
from ragcascade.datagen import synthetic_qa_dataset  # noqa: E402
from ragcascade.simulation import SessionState, dataset_to_corpus, next_query, RAMPS  # noqa: E402


def unit(rng, n, d):
    raw = rng.normal(size=(n, d))
    return (raw / np.linalg.norm(raw, axis=1, keepdims=True)).astype(np.float32)


def flat_index_cases():
    rng = np.random.default_rng(2024)
    out = {}
    cases = []
    specs = [(4, 3, 5), (8, 40, 12), (13, 200, 10), (64, 400, 10), (384, 300, 10), (768, 200, 5),
             (1024, 300, 10), (1024, 5, 10), (16, 1, 3)]
    for ci, (d, n, k) in enumerate(specs):
        X = unit(rng, n, d)
        if n >= 3:
            a, b, c = rng.choice(n, size=3, replace=False)
            X[b] = X[a]
            X[c] = X[a]
        else:
            a = 0
        Q = [unit(rng, 1, d)[0], X[int(a)].copy(), unit(rng, 1, d)[0]]
        idx = rc.FlatIndex(dim=d)
        for i in range(n):
            idx.insert(f"e{i}", X[i])
        rows = np.full((len(Q), k), -1, dtype=np.int64)
        scores = np.zeros((len(Q), k))
        count = np.zeros(len(Q), dtype=np.int32)
        for qi, q in enumerate(Q):
            hits = idx.search(q, k=k)
            count[qi] = len(hits)
            for j, h in enumerate(hits):
                rows[qi, j] = int(h.entry_id[1:])
                scores[qi, j] = h.score
        out[f"c{ci}_X"] = X
        out[f"c{ci}_Q"] = np.stack(Q).astype(np.float32)
        out[f"c{ci}_rows"] = rows
        out[f"c{ci}_scores"] = scores
        out[f"c{ci}_count"] = count
        cases.append({"name": f"c{ci}", "d": d, "n": n, "k": k})
    # orthogonal / one-hot (tests/test_index.py:44-49)
    X = np.eye(4, dtype=np.float32)[:2]
    idx = rc.FlatIndex(dim=4)
    idx.insert("e0", X[0])
    idx.insert("e1", X[1])
    hits = idx.search(np.eye(4, dtype=np.float32)[0], k=2)
    out["onehot_X"] = X
    out["onehot_Q"] = np.eye(4, dtype=np.float32)[:1]
    out["onehot_rows"] = np.array([[int(h.entry_id[1:]) for h in hits]], dtype=np.int64)
    out["onehot_scores"] = np.array([[h.score for h in hits]])
    out["onehot_count"] = np.array([len(hits)], dtype=np.int32)
    cases.append({"name": "onehot", "d": 4, "n": 2, "k": 2})
    np.savez_compressed(os.path.join(HERE, "flat_index.npz"), **out)
    return cases


def embed_cases():
    emb = rc.HashEmbedder()
    texts = ["what is the tallest mountain", "Who wrote Hamlet?", "alpha beta gamma", "gamma beta alpha",
             "!!!", "ünïcödé tokens ✓ here", "a", "x y x y", "The ledger0001 file for sector0001 in basin0001.",
             "What does the coastal ledger0007 report say about sector0007 near basin0007 cohort0007?"]
    out = []
    for t in texts:
        v = emb.embed(t).values
        nz = np.nonzero(v)[0]
        out.append({"text": t, "nz_index": nz.tolist(), "nz_value_bits": v[nz].view(np.uint32).tolist()})
    return out


def kv_cases():
    ops = []
    kv = rc.FixedKVCache(max_entries=3)

    def ans(t):
        return rc.AnswerRecord(text=t, layer=rc.LayerTag.MEMORY_RECALL, confidence=0.9)

    script = [("put", "a", "1"), ("put", "b", "2"), ("get", "a"), ("put", "c", "3"), ("put", "d", "4"),
              ("get", "a"), ("get", "b"), ("put", "b", "2b"), ("put", "e", "5"), ("get", "c"), ("get", "b"),
              ("get", "B"), ("get", "b "), ("put", "ü", "u"), ("get", "ü"), ("get", "d")]
    for op in script:
        if op[0] == "put":
            kv.put(op[1], ans(op[2]))
            ops.append({"op": "put", "key": op[1], "value": op[2], "len": len(kv)})
        else:
            got = kv.get(op[1])
            ops.append({"op": "get", "key": op[1], "result": got.text if got else None, "len": len(kv)})
    return {"max_entries": 3, "ops": ops, "stats": kv.stats(),
            "export": [e["query_text"] for e in kv.export_entries()]}


def router_trace():
    emb = rc.HashEmbedder()
    rows = synthetic_qa_dataset(300, seed=42)
    kb = rc.MainKnowledgeBase()
    rc.ingest_corpus((json.dumps(r) for r in dataset_to_corpus(rows[:60])), emb, kb=kb)
    router = rc.CascadeRouter(embedder=emb, backend=rc.StubBackend(), knowledge_base=kb)
    rng = np.random.default_rng([3, 0, 0])
    questions = [r["question"] for r in rows]
    state = SessionState("s1", questions, 200, RAMPS["linear"], 0.5)
    seq = []
    for _ in range(200):
        q, origin = next_query(state, rng)
        ans, ev = router.route(q)
        state.record_issued(q.text)
        seq.append({"text": q.text, "origin": origin,
                    "probes": [[p.layer.wire_name, p.outcome] for p in ev.layers_probed],
                    "serving": ev.serving_layer.wire_name, "answer": ans.text,
                    "passages": list(ans.supporting_passage_ids)})
    # a seeded-AKM probe: passage text identical to a later query (tests/test_router.py:152-167)
    router.adaptive_memory.settle()
    seeded = sorted(router.adaptive_memory.ids())[0]
    t = kb.get(seeded).text
    ans, ev = router.route(rc.validate_query(t, "s1"))
    seq.append({"text": t, "origin": "akm_probe", "probes": [[p.layer.wire_name, p.outcome] for p in ev.layers_probed],
                "serving": ev.serving_layer.wire_name, "answer": ans.text, "passages": list(ans.supporting_passage_ids)})
    st = router.stats()
    corpus = [{"id": c["id"], "text": c["text"], "source": c["source"], "answer": c["answer"]}
              for c in dataset_to_corpus(rows[:60])]
    return {"kb_rows": 60, "dataset_seed": 42, "dataset_n": 300, "corpus": corpus, "queries": seq,
            "stats": {"layer_counts": st["layer_counts"], "fixed_kv": st["fixed_kv"],
                      "semantic_cache": st["semantic_cache"], "adaptive_memory": st["adaptive_memory"],
                      "knowledge_base_searches": st["knowledge_base_searches"],
                      "sc_searches": router.semantic_cache.index.search_count,
                      "akm_searches": router.adaptive_memory.index.search_count,
                      "akm_inserted_total": router.adaptive_memory.inserted_total,
                      "context_calls": router.backend.context_calls, "recall_calls": router.backend.recall_calls}}


def simulation_logs():
    emb = rc.HashEmbedder()
    rows = synthetic_qa_dataset(400, seed=42)
    kb = rc.MainKnowledgeBase()
    rc.ingest_corpus((json.dumps(r) for r in dataset_to_corpus(rows)), emb, kb=kb)
    router = rc.CascadeRouter(embedder=emb, backend=rc.StubBackend(), knowledge_base=kb)
    logs = rc.run_simulation(rc.SimulationConfig(n_sessions=2, queries_per_session=150, seed=17), router, rows)
    return {"n_sessions": 2, "queries_per_session": 150, "seed": 17, "dataset_n": 400,
            "corpus": [{"id": c["id"], "text": c["text"], "source": c["source"], "answer": c["answer"]}
                       for c in dataset_to_corpus(rows)],
            "questions": [r["question"] for r in rows],
            "sessions": [list(log.to_jsonl_lines()) for log in logs]}


def snapshot_cases():
    import base64
    import struct
    import zlib

    rng = np.random.default_rng(77)
    d = 16
    idx = rc.FlatIndex(dim=d)
    X = unit(rng, 30, d)
    for i in range(30):
        idx.insert(f"doc-{i:03d}", X[i], {"n": i, "tag": "π" if i % 7 == 0 else "x"})
    # upserts keep their row: new vector + payload for two existing ids
    idx.insert("doc-004", X[20], {"n": 4, "tag": "upsert"})
    idx.insert("doc-011", unit(rng, 1, d)[0], None)
    Q = unit(rng, 4, d)
    Q[1] = X[20]
    snap = idx.snapshot()
    restored = rc.FlatIndex.restore(snap)

    def hits(ix):
        return [[(h.entry_id, h.score, h.rank) for h in ix.search(q, 5)] for q in Q]

    out = {"dim": d, "snapshot_b64": base64.b64encode(snap).decode(), "queries": Q.tolist(),
           "hits": hits(idx), "restored_hits": hits(restored),
           "restored_ids": list(restored.entry_ids()),
           "restored_payloads": [restored.payload(e) for e in restored.entry_ids()]}
    assert out["hits"] == out["restored_hits"]
    assert restored.snapshot() == snap

    header = struct.Struct("<8sIIQQI")

    def blob(vecs, recs, magic=b"RCFLATIX", version=1, crc_fix=0):
        meta = ("\n".join(json.dumps(r, ensure_ascii=False) for r in recs) + "\n").encode()
        body = np.asarray(vecs, dtype=np.float32).tobytes() + meta
        return header.pack(magic, version, d, len(recs), len(meta), zlib.crc32(body) ^ crc_fix) + body

    # duplicate id inside a snapshot: restore() upserts (the row stays, the last write wins)
    V = unit(rng, 6, d)
    recs = [{"id": f"k{i}", "payload": i} for i in range(6)]
    recs[4] = {"id": "k1", "payload": "second"}
    dup = blob(V, recs)
    rdup = rc.FlatIndex.restore(dup)
    out["dup_b64"] = base64.b64encode(dup).decode()
    out["dup_ids"] = list(rdup.entry_ids())
    out["dup_payloads"] = [rdup.payload(e) for e in rdup.entry_ids()]
    out["dup_hits"] = [[(h.entry_id, h.score, h.rank) for h in rdup.search(q, 6)] for q in V[:3]]
    out["dup_snapshot_b64"] = base64.b64encode(rdup.snapshot()).decode()
    # failures
    bad = {"bad_magic": blob(V, recs, magic=b"RCFLATIY"), "bad_version": blob(V, recs, version=2),
           "bad_crc": blob(V, recs, crc_fix=1), "short": dup[:20]}
    Vb = V.copy()
    Vb[2] *= 2.0
    bad["not_unit"] = blob(Vb, [{"id": f"k{i}", "payload": i} for i in range(6)])
    out["bad"] = {}
    for name, b in bad.items():
        try:
            rc.FlatIndex.restore(b)
            err = None
        except Exception as exc:  # noqa: BLE001
            err = type(exc).__name__
        out["bad"][name] = {"b64": base64.b64encode(b).decode(), "error": err}
    return out


def main():
    meta = {"flat_index_cases": flat_index_cases(), "numpy": np.__version__}
    with open(os.path.join(HERE, "flat_index.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    with open(os.path.join(HERE, "embed.json"), "w") as fh:
        json.dump(embed_cases(), fh, indent=1, ensure_ascii=False)
    with open(os.path.join(HERE, "kv_ops.json"), "w") as fh:
        json.dump(kv_cases(), fh, indent=1, ensure_ascii=False)
    with open(os.path.join(HERE, "router_trace.json"), "w") as fh:
        json.dump(router_trace(), fh, indent=1, ensure_ascii=False)
    with open(os.path.join(HERE, "simulation.json"), "w") as fh:
        json.dump(simulation_logs(), fh, ensure_ascii=False)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    if sys.argv[1:] == ["snapshot"]:
        with open(os.path.join(HERE, "snapshot.json"), "w") as fh:
            json.dump(snapshot_cases(), fh, indent=1, ensure_ascii=False)
    else:
        main()
