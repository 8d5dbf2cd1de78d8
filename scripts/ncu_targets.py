"""Small drivers for ncu captures of the non-tensor kernels.

    kv     100M-key table, 8 lookup batches of 65536 (fused fingerprint + probe)
    exact  fp64 einsum-order scan: 16 queries over 2M x 1024 (fallback / small-store path)
    embed  device HashEmbedder over 65536 workload texts
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

what = sys.argv[1]
torch.cuda.set_device(0)
if what == "kv":
    from benchlib.configs import c3_kv

    r = c3_kv(6538.6, n_keys=100_000_000, n_batches=8, steps=1)
    print({k: r[k] for k in ("value", "us_per_batch", "parity")})
elif what == "exact":
    import bench
    from paper_2506_21593_b200 import MODE_EXACT

    idx = bench.build_shard(2_000_000, 1024, 0, 2_000_000)
    q = bench.make_queries(2_000_000, 1024, 16)
    for _ in range(2):
        idx.search_batch(q, 10, mode=MODE_EXACT, validate=False)
    torch.cuda.synchronize()
    print("exact done")
elif what == "embed":
    from benchlib.workloads import qa_rows, session_stream
    from paper_2506_21593_b200 import HashEmbedder

    rows = qa_rows(120_000, 42)
    _, st = session_stream([r["question"] for r in rows], 65536, 0, 0)
    emb = HashEmbedder()
    for _ in range(2):
        v = emb.embed_device([t for t, _ in st])
    torch.cuda.synchronize()
    print("embed", tuple(v.shape))
