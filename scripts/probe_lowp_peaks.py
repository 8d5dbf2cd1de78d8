"""Measure cuBLAS(Lt) dense GEMM throughput for fp16, int8 (torch._int_mm) and
fp8 e4m3 (torch._scaled_mm) on the scan's shape (M=4096 queries x N rows x K=1024),
burst (best of 10) and sustained (back to back for ~4 s), with SM clocks.

Used to decide whether a lower-precision tensor-core scan pays under the
1000 W power cap, and as the int8 roofline denominator ("of measured").
"""
from __future__ import annotations

import json
import subprocess
import time

import torch


def sm_clock():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout.strip()
        return out
    except Exception:  # noqa: BLE001
        return "?"


def bench(fn, flop, secs=4.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    n = 0
    t0 = time.time()
    s.record()
    clk = None
    while time.time() - t0 < secs:
        for _ in range(8):
            fn()
        n += 8
        if clk is None and time.time() - t0 > secs / 2:
            clk = sm_clock()
    e.record()
    torch.cuda.synchronize()
    sus = s.elapsed_time(e) / n
    return flop / best / 1e9, flop / sus / 1e9, clk


def main():
    M, N, K = 4096, 65536, 1024
    res = {}
    a16 = torch.randn(M, K, device="cuda", dtype=torch.float16)
    b16 = torch.randn(N, K, device="cuda", dtype=torch.float16)
    flop = 2.0 * M * N * K
    res["fp16"] = bench(lambda: a16 @ b16.t(), flop)
    a8 = torch.randint(-127, 128, (M, K), device="cuda", dtype=torch.int8)
    b8 = torch.randint(-127, 128, (N, K), device="cuda", dtype=torch.int8)
    try:
        res["int8"] = bench(lambda: torch._int_mm(a8, b8.t()), flop)
    except Exception as ex:  # noqa: BLE001
        res["int8"] = repr(ex)
    try:
        af = a16.to(torch.float8_e4m3fn)
        bf = b16.to(torch.float8_e4m3fn)
        one = torch.ones((), device="cuda")
        res["fp8"] = bench(lambda: torch._scaled_mm(af, bf.t(), scale_a=one, scale_b=one, out_dtype=torch.float16), flop)
    except Exception as ex:  # noqa: BLE001
        res["fp8"] = repr(ex)
    for k, v in res.items():
        print(k, json.dumps(v))


if __name__ == "__main__":
    main()
