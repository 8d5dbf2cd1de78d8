"""Multi-rank sharded search on ONE GPU (both ranks on cuda:0, gloo carries the
all-gather of CUDA tensors): the row-sharded store + per-rank int8 scan + snap
flags + device merge must equal a single-index search bit for bit.

    torchrun --standalone --local-addr 127.0.0.1 --nproc-per-node 2 scripts/sharded_check.py
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2506_21593_b200 import MODE_TENSOR_I8  # noqa: E402
from paper_2506_21593_b200.sharded import ShardedFlatIndex, shard_range  # noqa: E402


def main():
    n, d, B = int(os.environ.get("N", "2000000")), 1024, 2048
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    lo, hi = shard_range(n, rank, world)
    idx = bench.build_shard(n, d, lo, hi)
    q = bench.make_queries(n, d, B)
    sh = ShardedFlatIndex(idx, lo)
    got = {}
    for k in (1, 5, 10):
        r = sh.search_batch(q, k)
        torch.cuda.synchronize()
        got[k] = (r.rows.cpu(), r.raw.cpu(), r.scores.cpu(), r.count.cpu())
    st = idx.stats()
    dist.barrier()
    if rank == 0:
        full = bench.build_shard(n, d, 0, n)
        bad = 0
        for k in (1, 5, 10):
            w = full.search_batch(q, k, mode=MODE_TENSOR_I8, validate=False)
            want = (w.rows.cpu(), w.raw.cpu(), w.scores.cpu(), w.count.cpu())
            for a, b_ in zip(got[k], want):
                bad += int((a != b_).sum().item())
        print(f"sharded world={world} rows/rank={hi - lo} local path={st.path} mismatches={bad}", flush=True)
        assert bad == 0
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
