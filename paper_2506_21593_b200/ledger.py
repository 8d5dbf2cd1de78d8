"""Columnar results of a routed batch, materialised into reference objects on demand.

A routed batch produces, per query, the serving layer, the answer text and
confidence, the supporting passages and a latency.  Building the
reference's ``AnswerRecord`` / ``RouteTraceEvent`` objects for every query
costs tens of microseconds of Python each, so ``route_batch`` records the
batch once as arrays (``BatchLedger``) and builds objects lazily — when the
caller asks for them, when the trace log is read, or when a cache entry
written by the batch is hit later (``LedgerEntry`` stands in for the
reference's ``CacheEntry``, caches.py:35-42).  Every materialised object is
identical to what sequential ``route`` would have produced.
"""
from __future__ import annotations

from functools import partial
from itertools import count, repeat
from operator import itemgetter
from typing import Sequence

import numpy as np

from .records import AnswerRecord, LayerTag, Query


class CtxRows:
    """j -> KB rows of query j's context passages (the first ``k`` of its retrieval
    top-k) for queries answered from retrieval, else None; sliced on access."""

    __slots__ = ("rows", "slot", "count", "k", "served")

    def __init__(self, rows: np.ndarray, slot: np.ndarray, count: np.ndarray, k: int, served: np.ndarray):
        self.rows, self.slot, self.count, self.k, self.served = rows, slot, count, k, served

    def get(self, j: int):
        if not self.served[j]:
            return None
        s = int(self.slot[j])
        return self.rows[s, : min(self.k, int(self.count[s]))]


class BatchLedger:
    __slots__ = ("queries", "layer", "latency", "text", "conf", "ctx_rows", "kb_index", "probe_prefix",
                 "_answers", "_events")

    def __init__(self, queries: Sequence[Query], layer: np.ndarray, latency: np.ndarray, text: list,
                 conf: np.ndarray, ctx_rows, kb_index, probe_prefix: dict):
        self.queries = queries          # the routed Query objects, in order
        self.layer = layer              # int8 [n] serving LayerTag value
        self.latency = latency          # float64 [n]
        self.text = text                # answer text per query
        self.conf = conf                # float64 [n] confidence
        self.ctx_rows = ctx_rows        # j -> KB rows of the context passages (L5 answers)
        self.kb_index = kb_index        # knowledge-base FlatIndex (passage payloads)
        self.probe_prefix = probe_prefix  # LayerTag -> tuple of LayerProbe before the serving probe
        self._answers: dict[int, AnswerRecord] = {}
        self._events: dict = {}

    def __len__(self) -> int:
        return len(self.queries)

    def passage_ids(self, j: int) -> tuple:
        rows = self.ctx_rows.get(j)
        if rows is None:
            return ()
        return tuple(self.kb_index.id_at(int(r)) for r in rows)

    def answer(self, j: int) -> AnswerRecord:
        a = self._answers.get(j)
        if a is None:
            a = AnswerRecord._trusted(self.text[j], LayerTag(int(self.layer[j])), float(self.conf[j]),
                                      self.passage_ids(j), float(self.latency[j]))
            self._answers[j] = a
        return a

    def event(self, j: int):
        ev = self._events.get(j)
        if ev is None:
            from .router import LayerProbe, RouteTraceEvent

            q = self.queries[j]
            L = LayerTag(int(self.layer[j]))
            lat = float(self.latency[j])
            probes = self.probe_prefix[L] + (LayerProbe(L, "hit", lat),)
            rows = self.ctx_rows.get(j)
            pairs = ()
            if rows is not None:
                pairs = tuple((self.kb_index.id_at(int(r)), self.kb_index.payload_at(int(r)).text) for r in rows)
            ev = RouteTraceEvent(q.id, q.session_id, q.text, probes, L, lat, q.issued_at, self.text[j], pairs)
            self._events[j] = ev
        return ev

    def results(self) -> list:
        return [(self.answer(j), self.event(j)) for j in range(len(self))]

    def layer_counts(self) -> dict[LayerTag, int]:
        vals, cnt = np.unique(self.layer, return_counts=True)
        return {LayerTag(int(v)): int(c) for v, c in zip(vals, cnt)}


class LedgerEntry(tuple):
    """A cache entry written by a routed batch; ``answer`` is built on first use.

    A tuple ``(query_text, ledger, j, created_at_ns)``: a span builds one per query, and
    ``entries_of`` makes them without running Python per entry (a class with ``__init__``
    cost ~0.3 us each, 1.2 ms per 4096-query span)."""

    __slots__ = ()

    def __new__(cls, query_text: str, ledger: BatchLedger, j: int, created_at_ns: int):
        return tuple.__new__(cls, (query_text, ledger, j, created_at_ns))

    query_text = property(itemgetter(0))
    _ledger = property(itemgetter(1))
    _j = property(itemgetter(2))
    created_at_ns = property(itemgetter(3))

    @property
    def answer(self) -> AnswerRecord:
        return self[1].answer(self[2])

    def text_conf(self) -> tuple[str, float]:
        lg, j = self[1], self[2]
        return lg.text[j], float(lg.conf[j])


_make_entry = partial(tuple.__new__, LedgerEntry)


def entries_of(texts: Sequence[str], ledger: BatchLedger, created_at_ns: int) -> list:
    """``[LedgerEntry(t, ledger, j, created_at_ns) for j, t in enumerate(texts)]``, built in C."""
    return list(map(_make_entry, zip(texts, repeat(ledger), count(), repeat(created_at_ns))))


def entry_text_conf(entry) -> tuple[str, float]:
    """(answer text, confidence) of a CacheEntry or LedgerEntry without materialising."""
    if isinstance(entry, LedgerEntry):
        return entry.text_conf()
    a = entry.answer
    return a.text, a.confidence
