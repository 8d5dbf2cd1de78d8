"""Texts -> one UTF-8 byte arena + int64 offsets (the device-side text format)."""
from __future__ import annotations

from typing import Sequence

import numpy as np


def encode_texts(texts: Sequence[str]):
    """(bytes uint8 [total], offsets int64 [n+1]) as host numpy arrays.
    ``surrogatepass`` keeps the str -> bytes map injective for every Python str."""
    joined = "".join(texts)
    if joined.isascii():  # one byte per character: no per-text encode
        off = np.zeros(len(texts) + 1, dtype=np.int64)
        if texts:
            np.cumsum(np.fromiter(map(len, texts), dtype=np.int64, count=len(texts)), out=off[1:])
        return np.frombuffer(joined.encode("ascii") or b"\0", dtype=np.uint8).copy(), off
    bs = [t.encode("utf-8", "surrogatepass") for t in texts]
    off = np.zeros(len(bs) + 1, dtype=np.int64)
    if bs:
        np.cumsum([len(b) for b in bs], out=off[1:])
    data = np.frombuffer(b"".join(bs) or b"\0", dtype=np.uint8).copy()
    return data, off


class DeviceTexts(tuple):
    """(data, offsets) device tensors of a text arena, unpackable as a pair; ``nbytes``
    (the arena's byte count) and ``n`` (texts) stay on the host so callers never read
    them back from the device."""

    def __new__(cls, data, off, host_off):
        t = super().__new__(cls, (data, off))
        t.host_off = host_off
        t.n = len(host_off) - 1
        t.nbytes = int(host_off[-1])
        t.ascii = None  # True when every text is ASCII (one byte per character), if known
        return t

    def nbytes_of(self, n: int) -> int:
        """bytes of the first ``n`` texts"""
        return int(self.host_off[n])


def to_device(texts: Sequence[str]) -> DeviceTexts:
    from ._lib import h2d

    data, off = encode_texts(texts)
    t = DeviceTexts(h2d(data), h2d(off), off)
    # UTF-8 spends >= 2 bytes on every non-ASCII character (and surrogatepass 3 on a surrogate)
    t.ascii = sum(map(len, texts)) == t.nbytes
    return t
