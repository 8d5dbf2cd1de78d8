"""Small end-to-end run of every device path, for compute-sanitizer (memcheck /
racecheck / synccheck): int8, fp16 and exact searches with row limits, KV put/get,
the device embedder and a short routed batch."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_21593_b200 import MODE_EXACT, MODE_TENSOR, MODE_TENSOR_I8, FlatIndex, FixedKVCache  # noqa: E402
from paper_2506_21593_b200 import HashEmbedder  # noqa: E402


def main():
    rng = np.random.default_rng(1)
    n, d = int(os.environ.get("N", "20000")), 256
    X = rng.standard_normal((n, d)).astype(np.float32)
    X = (X / np.linalg.norm(X.astype(np.float64), axis=1, keepdims=True)).astype(np.float32)
    idx = FlatIndex(dim=d)
    idx.extend_arrays([f"r{i}" for i in range(n)], X)
    Q = X[rng.integers(0, n, 300)] + 0.01 * rng.standard_normal((300, d)).astype(np.float32)
    Q = (Q / np.linalg.norm(Q.astype(np.float64), axis=1, keepdims=True)).astype(np.float32)
    lim = rng.integers(1, n + 1, 300)
    for mode in (MODE_TENSOR_I8, MODE_TENSOR, MODE_EXACT):
        for k in (1, 10):
            a = idx.search_batch(Q, k, mode=mode, validate=False)
            b = idx.search_batch(Q, k, mode=mode, validate=False, row_limit=lim)
            torch.cuda.synchronize()
            print("mode", mode, "k", k, int(a.count.sum()), int(b.count.sum()), flush=True)
    kv = FixedKVCache()
    from paper_2506_21593_b200.caches import CacheEntry  # noqa: F401

    texts = [f"query-{i:09d}" for i in range(5000)]
    emb = HashEmbedder(dim=d)
    V = emb.embed_device(texts)
    torch.cuda.synchronize()
    print("embed", tuple(V.shape), flush=True)
    from paper_2506_21593_b200.textarena import to_device

    dd, do = to_device(texts)
    vals, hit = kv.probe_device(dd, do, len(texts))
    torch.cuda.synchronize()
    print("kv probe", int(hit.sum().item()), flush=True)


if __name__ == "__main__":
    main()
