"""cudaMalloc / cudaFree / cudaMallocAsync costs on the box, with a large resident store."""
import ctypes
import time

import torch

rt = ctypes.CDLL("libcudart.so.12") if False else None
try:
    from cuda.bindings import runtime as cr
except ImportError:
    from cuda import cudart as cr


def t_malloc(nbytes, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        err, p = cr.cudaMalloc(nbytes)
        t1 = time.perf_counter()
        cr.cudaFree(p)
        t2 = time.perf_counter()
        out.append(((t1 - t) * 1e3, (t2 - t1) * 1e3))
    return out


def t_async(nbytes, reps=3):
    out = []
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        err, p = cr.cudaMallocAsync(nbytes, s)
        cr.cudaFreeAsync(p, s)
        cr.cudaStreamSynchronize(s)
        out.append((time.perf_counter() - t) * 1e3)
    return out


for label in ("empty", "with 100 GB resident"):
    if label != "empty":
        big = [torch.empty(10 * 2**30, dtype=torch.uint8, device="cuda") for _ in range(10)]
    for mb in (8, 64, 256, 1024, 4096):
        print(label, f"{mb} MB malloc/free ms:", [(round(a, 2), round(b, 2)) for a, b in t_malloc(mb << 20)],
              "async:", [round(x, 2) for x in t_async(mb << 20)], flush=True)
