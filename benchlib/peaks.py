"""In-run int8 tensor peak: MEASURED_PEAKS.json (driver-written) has the bf16 peaks
only, so the int8 denominator is measured here with the driver's own method applied
to int8: cuBLAS(Lt) int8 GEMM (torch._int_mm) at 8192^3, best of 10 (burst) and back
to back for `seconds` (sustained, under the power cap)."""
from __future__ import annotations

import time

_CACHE: dict = {}


def int8_peak(seconds: float = 3.0) -> dict:
    if "int8" in _CACHE:
        return _CACHE["int8"]
    import torch

    n = 8192
    a = torch.randint(-127, 128, (n, n), device="cuda", dtype=torch.int8)
    b = torch.randint(-127, 128, (n, n), device="cuda", dtype=torch.int8).t()  # column-major operand
    ops = 2.0 * n * n * n
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        s.record()
        torch._int_mm(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    it = 0
    t0 = time.time()
    s.record()
    while time.time() - t0 < seconds:
        for _ in range(8):
            torch._int_mm(a, b)
        it += 8
    e.record()
    torch.cuda.synchronize()
    sus = s.elapsed_time(e) / it
    out = {"int8_tops": ops / best / 1e9, "int8_tops_sustained": ops / sus / 1e9,
           "how": f"torch._int_mm int8 {n}^3 (2*N^3 ops): best of 10 (burst), back to back for {seconds:g} s "
                  f"(sustained), measured in this run"}
    del a, b
    torch.cuda.empty_cache()
    _CACHE["int8"] = out
    return out
