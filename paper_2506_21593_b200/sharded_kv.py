"""Fixed-KV table hash-partitioned across ranks (one process per GPU).

Rank r owns the keys whose 128-bit fingerprint satisfies ``fp_lo % world == r``
(the low word is independent of the bucket bits the table probes with).  A
put inserts only the owned keys of the batch; a lookup probes the whole batch
on every rank — keys a rank does not own simply miss there (value -1) — and
ONE all-reduce(max) over the int64 values combines them: the owner reports the
key's write sequence number (>= 0), everyone else -1.  Byte-exact semantics
are those of ``FixedKVCache`` (caches.py:57-77); last-write-wins still holds
because a key lives on exactly one rank.

The probe and combine are injectable so the plumbing runs on CPU with gloo.
"""
from __future__ import annotations

import ctypes
from typing import Callable

from . import _lib
from .textarena import encode_texts


class ShardedKV:
    def __init__(self, capacity: int = 1024, *, group=None, probe: Callable | None = None,
                 insert: Callable | None = None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self._probe = probe
        self._insert = insert
        self._h = None
        if probe is None or insert is None:
            _lib.require_device()
            L = _lib.load()
            h = ctypes.c_void_p()
            _lib.check(L.pr_kv_create(max(1024, capacity // max(1, self.world)), ctypes.byref(h)), "kv_create")
            self._h = h

    # production path -------------------------------------------------------
    def _fingerprints(self, texts):
        import torch

        data, off = encode_texts(texts)
        d_data, d_off = torch.from_numpy(data).cuda(), torch.from_numpy(off).cuda()
        fp = torch.empty((len(texts), 2), dtype=torch.int64, device="cuda")
        L = _lib.load()
        _lib.check(L.pr_fingerprint(_lib.ptr(d_data), _lib.ptr(d_off), len(texts), _lib.ptr(fp), _lib.stream_ptr()),
                   "fingerprint")
        return fp

    def owner(self, fp):
        """Owning rank of each fingerprint (int64 [n, 2] tensor)."""
        lo = fp[:, 1]
        return (lo.remainder(self.world) + self.world).remainder(self.world)  # non-negative modulo

    def put(self, texts, values) -> int:
        """Insert the keys this rank owns; ``values`` are int64 write sequence numbers."""
        import torch

        fp = self._fingerprints(texts) if self._insert is None else None
        vals = torch.as_tensor(values, dtype=torch.int64)
        if self._insert is not None:
            return self._insert(texts, vals, self.rank, self.world)
        vals = vals.cuda()
        mine = self.owner(fp) == self.rank
        fp_m, v_m = fp[mine].contiguous(), vals[mine].contiguous()
        L = _lib.load()
        if fp_m.shape[0]:
            _lib.check(L.pr_kv_put(self._h, _lib.ptr(fp_m), _lib.ptr(v_m), fp_m.shape[0], _lib.stream_ptr()), "put")
        return int(fp_m.shape[0])

    def get(self, texts):
        """(values int64 [n], hit bool [n]) for every key, combined over ranks."""
        import torch
        import torch.distributed as dist

        if self._probe is not None:
            vals = self._probe(texts, self.rank, self.world)
        else:
            data, off = encode_texts(texts)
            d_data, d_off = torch.from_numpy(data).cuda(), torch.from_numpy(off).cuda()
            vals = torch.empty(len(texts), dtype=torch.int64, device="cuda")
            hit = torch.empty(len(texts), dtype=torch.uint8, device="cuda")
            L = _lib.load()
            _lib.check(L.pr_kv_get_text(self._h, _lib.ptr(d_data), _lib.ptr(d_off), len(texts), _lib.ptr(vals),
                                        _lib.ptr(hit), _lib.stream_ptr()), "get")
        if self.world > 1:
            dist.all_reduce(vals, op=dist.ReduceOp.MAX, group=self.group)
        return vals, vals >= 0
