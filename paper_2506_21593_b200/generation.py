"""Generation-side collaborators of the router (LLM stubbed).

Restates the parts of ``ragcascade/generation.py`` the cascade calls:
``StubKnowledgeTable``/``StubBackend`` (:51-115), ``generate_with_context``
(:178-200), ``memory_recall`` (:203-224) and ``answer_with_latency``.  The
LLM itself is out of scope; any object with the reference's
``generate_with_context(query_text, passages)`` / ``recall(query_text)``
methods can be plugged in.
"""
from __future__ import annotations

import re
from dataclasses import replace
from typing import Protocol, Sequence

from .errors import EmptyContext
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
