"""Pinned staging ring for host<->device copies on the cascade's pipelined path.

``torch.empty(pin_memory=True)`` / ``Tensor.pin_memory()`` allocate page-locked memory per
call (measured 3.9 ms per call inside a pipelined route_batch span), and a copy from
pageable memory makes the host wait for the device.  One process-wide ring of pinned
memory serves every small upload and read-back instead: a copy takes the next region,
records an event after the copy, and a region is reused only once its event has
completed (the ring is large enough that this never waits in practice).
"""
from __future__ import annotations

import collections
import threading

import numpy as np

_ALIGN = 256


class PinnedRing:
    def __init__(self, nbytes: int = 64 << 20):
        import torch

        self.cap = int(nbytes)
        self.buf = torch.empty(self.cap, dtype=torch.uint8, pin_memory=True)
        self.arr = self.buf.numpy()
        self.head = 0
        self.live: collections.deque = collections.deque()  # (start, end, event), allocation order
        self.lock = threading.Lock()

    def _take(self, nbytes: int) -> int:
        """Start offset of a free region of ``nbytes`` (caller holds the lock)."""
        nb = (nbytes + _ALIGN - 1) // _ALIGN * _ALIGN
        a = self.head if self.head + nb <= self.cap else 0
        b = a + nb
        while self.live:
            s, e, ev = self.live[0]
            if ev.query():
                self.live.popleft()
                continue
            break
        for s, e, ev in list(self.live):
            if s < b and a < e:  # an in-flight region still covers part of this one
                ev.synchronize()
        while self.live and self.live[0][2].query():
            self.live.popleft()
        self.head = b
        return a

    def h2d(self, x: np.ndarray):
        """Device copy of host array ``x`` (queued on the current stream, host returns at once)."""
        import torch

        x = np.ascontiguousarray(x)
        nb = x.nbytes
        dev = torch.empty(x.shape, dtype=_TORCH_OF[x.dtype.str], device="cuda")
        if nb == 0:
            return dev
        with self.lock:
            a = self._take(nb)
            self.arr[a:a + nb] = x.reshape(-1).view(np.uint8)
            dev.view(-1).view(torch.uint8).copy_(self.buf[a:a + nb], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self.live.append((a, a + nb, ev))
        return dev

    def d2h(self, t):
        """(host numpy view, event): ``t`` copied into the ring on the current stream; read the
        view after ``event.synchronize()`` and copy out what must outlive the next wrap."""
        import torch

        t = t.contiguous()
        nb = t.numel() * t.element_size()
        with self.lock:
            a = self._take(max(nb, 1))
            self.buf[a:a + nb].copy_(t.view(-1).view(torch.uint8), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self.live.append((a, a + max(nb, 1), ev))
        view = self.arr[a:a + nb].view(_NUMPY_OF[t.dtype]).reshape(tuple(t.shape))
        return view, ev


def _dtype_maps():
    import torch

    tn = {np.dtype(np.uint8).str: torch.uint8, np.dtype(np.int8).str: torch.int8,
          np.dtype(np.int32).str: torch.int32, np.dtype(np.int64).str: torch.int64,
          np.dtype(np.float32).str: torch.float32, np.dtype(np.float64).str: torch.float64,
          np.dtype(np.bool_).str: torch.bool}
    nt = {v: np.dtype(k) for k, v in tn.items()}
    return tn, nt


class _Lazy(dict):
    def __init__(self, which):
        super().__init__()
        self.which = which

    def __missing__(self, key):
        tn, nt = _dtype_maps()
        self.update(tn if self.which == 0 else nt)
        return dict.__getitem__(self, key)


_TORCH_OF = _Lazy(0)
_NUMPY_OF = _Lazy(1)

_ring: PinnedRing | None = None
_ring_lock = threading.Lock()


def ring() -> PinnedRing:
    global _ring
    if _ring is None:
        with _ring_lock:
            if _ring is None:
                _ring = PinnedRing()
    return _ring
