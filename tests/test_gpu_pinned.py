"""The pinned staging ring (pinned.py) behind every small upload / read-back of the pipelined
cascade: copies land intact across ring wrap-arounds while earlier copies are still queued
behind device work, and the host never reads a region before its copy completed."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_ring_h2d_wraps_under_queued_work(gpu):
    import torch

    from paper_2506_21593_b200.pinned import PinnedRing

    r = PinnedRing(1 << 20)
    rng = np.random.default_rng(0)
    a = torch.randn(4096, 4096, device="cuda")
    sent, got = [], []
    for i in range(300):
        if i % 50 == 0:
            a = a @ a  # keep the stream busy so earlier copies are still pending at wrap time
            a /= a.norm()
        x = rng.integers(-2**40, 2**40, size=int(rng.integers(1, 20000)), dtype=np.int64)
        sent.append(x)
        got.append(r.h2d(x))
    torch.cuda.synchronize()
    for x, d in zip(sent, got):
        assert (d.cpu().numpy() == x).all()


@pytest.mark.parametrize("dtype", ["int64", "int32", "uint8", "float32", "float64", "bool"])
def test_ring_round_trip_dtypes(gpu, dtype):
    import torch

    from paper_2506_21593_b200 import _lib
    from paper_2506_21593_b200.pinned import ring

    rng = np.random.default_rng(1)
    x = (rng.random(12345) > 0.5) if dtype == "bool" else (rng.random(12345) * 1000).astype(dtype)
    d = _lib.h2d(x)
    assert d.is_cuda and str(d.dtype) == f"torch.{dtype}"
    view, ev = ring().d2h(d * 1 if dtype != "bool" else d.clone())
    ev.synchronize()
    assert (view == x).all()
    assert (d.cpu().numpy() == x).all()
    # dtype conversion on the way in
    d64 = _lib.h2d(np.arange(10, dtype=np.int32), torch.int64)
    assert d64.dtype == torch.int64 and d64.cpu().tolist() == list(range(10))
