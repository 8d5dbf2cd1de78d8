"""Fixed-KV table hash-partitioned across ranks (one process per GPU).

Rank r owns the keys whose hash maps to r: ``owner = (tag & 0x7fffffff) % world`` where
tag is the key's 32-bit tag hash (``owner_host`` / device ``pr_kv_owner``).  The table's
home slot comes from the OTHER, independent hash chain, so the ownership bits and the
slot bits are disjoint: every slot of a rank's table is a home slot for its keys
(round 1 took both from the same low bits, so at world 8 only 1/8 of a rank's buckets
could be home buckets).

A put inserts only the keys a rank owns; a lookup runs ``pr_kv_get_text_owned`` on every
rank over the whole (broadcast) batch, which hashes each key once and probes only the
owned ones — per-rank probe traffic is ~B/world — and ONE all-reduce(max) over the int64
values combines them: the owner reports the key's write sequence number (>= 0), everyone
else -1.  Byte-exact semantics are those of ``FixedKVCache`` (caches.py:57-77);
last-write-wins still holds because a key lives on exactly one rank.

The probe and insert are injectable so the plumbing runs on CPU with gloo.
"""
from __future__ import annotations

import ctypes
from typing import Callable

from . import _lib
from .textarena import to_device


def owner_host(text: str, world: int) -> int:
    """Owning rank of ``text`` (host twin of the device ``owner_of``, kv.cu)."""
    from .caches import fingerprint_host

    tag = fingerprint_host(text)[0]
    return (tag & 0x7FFFFFFF) % world


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

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().pr_kv_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None

    def owners(self, arena):
        """Owning rank of every key of a ``DeviceTexts`` arena (int32 device tensor)."""
        import torch

        own = torch.empty(arena.n, dtype=torch.int32, device="cuda")
        if arena.n:
            _lib.check(_lib.load().pr_kv_owner(_lib.ptr(arena[0]), _lib.ptr(arena[1]), arena.n, self.world,
                                               _lib.ptr(own), _lib.stream_ptr()), "kv_owner")
        return own

    def put(self, texts, values) -> None:
        """Insert the keys this rank owns; ``values`` are int64 write sequence numbers."""
        import torch

        vals = torch.as_tensor(values, dtype=torch.int64)
        if self._insert is not None:
            self._insert(texts, vals, self.rank, self.world)
            return
        arena = to_device(texts)
        vals = vals.cuda()
        _lib.check(_lib.load().pr_kv_put_text_owned(self._h, _lib.ptr(arena[0]), _lib.ptr(arena[1]), arena.n,
                                                    arena.nbytes, _lib.ptr(vals), self.rank, self.world,
                                                    _lib.stream_ptr()), "kv_put")

    def get_arena(self, arena):
        """(values int64 [n], hit bool [n]) for a device text arena, combined over ranks."""
        import torch
        import torch.distributed as dist

        vals = torch.empty(arena.n, dtype=torch.int64, device="cuda")
        hit = torch.empty(arena.n, dtype=torch.uint8, device="cuda")
        _lib.check(_lib.load().pr_kv_get_text_owned(self._h, _lib.ptr(arena[0]), _lib.ptr(arena[1]), arena.n,
                                                    self.rank, self.world, _lib.ptr(vals), _lib.ptr(hit),
                                                    _lib.stream_ptr()), "kv_get")
        if self.world > 1:
            dist.all_reduce(vals, op=dist.ReduceOp.MAX, group=self.group)
        return vals, vals >= 0

    def get(self, texts):
        """(values int64 [n], hit bool [n]) for every key, combined over ranks."""
        import torch.distributed as dist

        if self._probe is None:
            return self.get_arena(to_device(texts))
        vals = self._probe(texts, self.rank, self.world)
        if self.world > 1:
            dist.all_reduce(vals, op=dist.ReduceOp.MAX, group=self.group)
        return vals, vals >= 0
