"""Generation-side collaborators of the router (LLM stubbed).

Restates the parts of ``ragcascade/generation.py`` the cascade calls:
``StubKnowledgeTable``/``StubBackend`` (:51-115), ``generate_with_context``
(:178-200), ``memory_recall`` (:203-224) and ``answer_with_latency``.  The
LLM itself is out of scope; any object with the reference's
``generate_with_context(query_text, passages)`` / ``recall(query_text)``
methods can be plugged in.

``DeviceKnowledgeTable`` is the L3 recall table on the GPU: a
``StubKnowledgeTable`` drop-in kept in a second instance of the fixed-KV hash
table (byte-exact question keys, value = index of the (answer, confidence)
entry), so a routed batch decides L3 on the device (``pr_recall_gate``) and
hands the outcome to the cascade gate with L1/L2.
"""
from __future__ import annotations

import json
import re
from dataclasses import dataclass, replace
from typing import Iterable, Protocol, Sequence

from .errors import EmptyContext, MalformedJsonl
from .records import AnswerRecord, LayerTag, Passage, Query

STUB_CONFIDENCE = 0.9
DEFAULT_RECALL_THRESHOLD = 0.5
_SENTENCE_END = re.compile(r"(?<=[.!?])\s+")


def first_sentence(text: str) -> str:
    head = _SENTENCE_END.split(text.strip(), maxsplit=1)
    return head[0] if head and head[0] else text.strip()


class GenerationBackend(Protocol):
    def generate_with_context(self, query_text: str, passages: Sequence[Passage]) -> tuple[str, float]: ...

    def recall(self, query_text: str) -> tuple[str, float]: ...


class StubKnowledgeTable:
    """Exact question -> (answer, confidence)."""

    def __init__(self) -> None:
        self._table: dict[str, tuple[str, float]] = {}

    def add(self, question: str, answer: str, confidence: float = STUB_CONFIDENCE) -> None:
        if not 0.0 <= confidence <= 1.0:
            raise ValueError(f"confidence {confidence} outside [0, 1]")
        self._table[question] = (answer, confidence)

    def lookup(self, question: str) -> tuple[str, float] | None:
        return self._table.get(question)

    def __len__(self) -> int:
        return len(self._table)

    @classmethod
    def from_triples_jsonl(cls, path, confidence: float = STUB_CONFIDENCE) -> "StubKnowledgeTable":
        table = cls()
        for o in _read_triples(path):
            table.add(str(o["question"]), str(o["answer"]), confidence)
        return table


def _read_triples(path) -> list[dict]:
    """Strict JSONL reader of ``ragcascade/jsonl.py:12-49`` (blank lines skipped, a
    malformed line or a non-object raises MalformedJsonl with its 1-based number)."""
    out = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line:
                continue
            try:
                obj = json.loads(line)
            except json.JSONDecodeError as exc:
                raise MalformedJsonl(f"line {lineno}: {exc}", line_number=lineno) from exc
            if not isinstance(obj, dict):
                raise MalformedJsonl(f"line {lineno}: expected a JSON object, got {type(obj).__name__}",
                                     line_number=lineno)
            out.append(obj)
    return out


@dataclass(frozen=True)
class RecallEntry:
    answer: str
    confidence: float


class DeviceKnowledgeTable:
    """``StubKnowledgeTable`` (generation.py:51-80) on the GPU: exact question text ->
    (answer, confidence) in a fixed-KV device table (``caches.FixedKVCache``: byte-exact
    keys, the latest ``add`` of a question wins).  ``lookup`` probes the device (what
    ``StubBackend.recall`` calls per query); ``gate_device`` is the batched L3 decision of
    ``memory_recall`` (generation.py:203-224) for a routed span, on the device."""

    def __init__(self, *, capacity: int = 1024):
        from .caches import FixedKVCache

        self._kv = FixedKVCache(capacity=capacity)
        self._conf_d = None  # device float64 [arena]: confidence, -1 where the answer is empty

    @staticmethod
    def _check(confidence: float) -> float:
        if not 0.0 <= confidence <= 1.0:
            raise ValueError(f"confidence {confidence} outside [0, 1]")
        return confidence

    def add(self, question: str, answer: str, confidence: float = STUB_CONFIDENCE) -> None:
        self.add_many([question], [answer], [confidence])

    def add_many(self, questions: Sequence[str], answers: Sequence[str],
                 confidences: Iterable[float] | float = STUB_CONFIDENCE) -> None:
        """Bulk ``add`` in order (a later add of a question wins); every confidence is
        validated before anything is inserted."""
        if isinstance(confidences, (int, float)):
            confidences = [confidences] * len(questions)
        confs = [self._check(c) for c in confidences]
        if not (len(questions) == len(answers) == len(confs)):
            raise ValueError("questions, answers and confidences differ in length")
        if not questions:
            return
        self._kv.put_entries(list(questions), [RecallEntry(a, c) for a, c in zip(answers, confs)])
        self._conf_d = None  # rebuilt from the (possibly compacted) arena on the next gate

    def lookup(self, question: str) -> tuple[str, float] | None:
        from .textarena import to_device

        arena = to_device([question])
        with self._kv._lock:
            vals, hit = self._kv.probe_device(arena[0], arena[1], 1)
            if not int(hit.item()):
                return None
            e = self._kv.entry_at(int(vals.item()))
        return e.answer, e.confidence

    def entry_at(self, value: int) -> RecallEntry:
        return self._kv.entry_at(value)

    def __len__(self) -> int:
        return len(self._kv)

    def __bool__(self) -> bool:
        # StubBackend replaces a falsy table (``knowledge or StubKnowledgeTable()``,
        # generation.py:95): an empty device table must stay the table
        return True

    def _device_conf(self):
        import torch

        if self._conf_d is None:
            arena = self._kv._arena
            c = [e.confidence if e.answer else -1.0 for e in arena] or [-1.0]
            self._conf_d = torch.tensor(c, dtype=torch.float64).cuda()
        return self._conf_d

    def gate_device(self, d_data, d_off, n: int, threshold: float):
        """L3 for a batch of ``n`` question texts (device UTF-8 arena): (values int64 [n],
        accepted uint8 [n]) device tensors; accepted iff found, confidence >= threshold and
        the answer is non-empty.  Nothing is read back."""
        import torch

        from . import _lib

        with self._kv._lock:
            vals, hit = self._kv.probe_device(d_data, d_off, n)
            conf = self._device_conf()
            out = torch.empty(n, dtype=torch.uint8, device="cuda")
            _lib.check(_lib.load().pr_recall_gate(n, _lib.ptr(vals), _lib.ptr(hit), _lib.ptr(conf), conf.numel(),
                                                  float(threshold), _lib.ptr(out), _lib.stream_ptr()), "recall_gate")
        return vals, out

    @classmethod
    def from_triples_jsonl(cls, path, confidence: float = STUB_CONFIDENCE) -> "DeviceKnowledgeTable":
        objs = _read_triples(path)
        table = cls(capacity=max(1024, 2 * len(objs)))
        table.add_many([str(o["question"]) for o in objs], [str(o["answer"]) for o in objs], confidence)
        return table


class StubBackend:
    """Context mode answers with the top passage's annotation (or its first
    sentence); recall consults the table, unknown questions get confidence 0."""

    def __init__(self, knowledge: StubKnowledgeTable | None = None, context_confidence: float = STUB_CONFIDENCE):
        self.knowledge = knowledge or StubKnowledgeTable()
        self.context_confidence = context_confidence
        self.context_calls = 0
        self.recall_calls = 0

    def generate_with_context(self, query_text: str, passages: Sequence[Passage]) -> tuple[str, float]:
        self.context_calls += 1
        top = passages[0]
        return (top.answer if top.answer else first_sentence(top.text)), self.context_confidence

    def recall(self, query_text: str) -> tuple[str, float]:
        self.recall_calls += 1
        return self.knowledge.lookup(query_text) or ("", 0.0)


def generate_with_context(backend, query: Query, passages: Sequence[Passage], layer: LayerTag) -> AnswerRecord:
    if layer not in (LayerTag.ADAPTIVE_MEMORY, LayerTag.NAIVE_RAG):
        raise ValueError(f"context generation cannot serve layer {layer.wire_name}")
    if not passages:
        raise EmptyContext("context generation requires at least one passage")
    text, conf = backend.generate_with_context(query.text, passages)
    return AnswerRecord(text=text, layer=layer, confidence=conf,
                        supporting_passage_ids=tuple(p.id for p in passages), latency_seconds=0.0)


def memory_recall(backend, query: Query, recall_threshold: float = DEFAULT_RECALL_THRESHOLD) -> AnswerRecord | None:
    if not 0.0 <= recall_threshold <= 1.0:
        raise ValueError(f"recall_threshold {recall_threshold} outside [0, 1]")
    text, conf = backend.recall(query.text)
    if conf < recall_threshold or not text:
        return None
    return AnswerRecord(text=text, layer=LayerTag.MEMORY_RECALL, confidence=conf, supporting_passage_ids=(),
                        latency_seconds=0.0)


def answer_with_latency(answer: AnswerRecord, latency_seconds: float) -> AnswerRecord:
    return replace(answer, latency_seconds=latency_seconds)
