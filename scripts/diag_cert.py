"""Why do sparse (HashEmbedder) queries fail the tcgen05 certificate on the C5 KB?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from benchlib.workloads import corpus_of, qa_rows, session_stream  # noqa: E402
from paper_2506_21593_b200 import HashEmbedder, MODE_TENSOR  # noqa: E402

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
idx = bench.build_shard(n, 1024, 0, n)
emb = HashEmbedder()
rows = qa_rows(120_000, 42)
ctx = emb.embed_matrix([c["text"] for c in corpus_of(rows)])
idx._update_rows(np.arange(120_000, dtype=np.int64), ctx)
_, st = session_stream([r["question"] for r in rows], 4096, 0, 0)
Q = torch.from_numpy(emb.embed_matrix([t for t, _ in st])).cuda()
res = idx.search_batch(Q, 10, mode=MODE_TENSOR, validate=False)
s = idx.stats()
print("queries", s.queries, "fallback", s.fallback, "nsplit(last exact)", s.nsplit)
X16 = None
# exact + approx scores for a few queries, on the GPU with torch (diagnostic only)
X = idx.read_rows(0, n)
Xh = X.half()
E = 1.11e-3
fails = 0
for qi in range(0, 400):
    q = Q[qi]
    ex = (X.double() @ q.double())
    ap = (Xh.float() @ q.half().float())
    top_ex = torch.topk(ex, 12)
    top_ap = torch.topk(ap, 12)
    gap = (top_ex.values[9] - top_ex.values[10]).item()
    nnz = int((q != 0).sum())
    if qi < 20 or gap < 3e-3:
        print(f"q{qi} nnz={nnz} e1={top_ex.values[0]:.4f} e10={top_ex.values[9]:.5f} e11={top_ex.values[10]:.5f} "
              f"a10={top_ap.values[9]:.5f} maxerr={float((ex - ap.double()).abs().max()):.2e} "
              f"rows={top_ex.indices[:10].tolist()}")
