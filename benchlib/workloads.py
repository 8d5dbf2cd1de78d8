"""Workload generators for the C1/C5 replays (bench and test infrastructure).

Restatements, from the reference's behaviour, of the pieces that generate
PentaRAG's nine-session cache-warming workload — they are NOT on the hot path
and nothing in paper_2506_21593_b200 imports them:

* ``qa_rows``            ~ ragcascade/datagen.py:51-72 (synthetic_qa_dataset)
* ``mutate``             ~ ragcascade/simulation.py:102-135 (perturb)
* ``Session.draw``       ~ ragcascade/simulation.py:241-265 (next_query)
* ``LatencyDraws``       ~ ragcascade/metrics.py:440-466 (SyntheticLatencyModel)
* ``simulate_batched``   ~ ragcascade/simulation.py:268-314 (run_simulation),
  routing each session with ``route_batch`` and re-timing the events after
  the fact (query texts never depend on routing outcomes, only timestamps do)

Same RNG call order as the reference, so the same seeds give the same
streams; tests/test_workloads.py pins them to the reference's recorded
simulation logs.
"""
from __future__ import annotations

import dataclasses
import json
from typing import Callable, Sequence

import numpy as np

# question shapes: one shared adjective slot + four row-unique tokens
_SHAPES = (
    "What does the {a} {b} report say about {c} near {d} {e}?",
    "Which {a} {b} facility processed {c} shipments for {d} {e}?",
    "Who maintains the {a} {b} registry covering {c} under {d} {e}?",
    "When was the {a} {b} survey of {c} completed for {d} {e}?",
    "Where is the {a} {b} archive for {c} stored inside {d} {e}?",
    "How often does the {a} {b} audit review {c} within {d} {e}?",
)
_ADJ = ("coastal", "northern", "annual", "regional", "municipal", "federated",
        "seasonal", "upstream", "granite", "maritime", "orbital", "alpine")
_LEAD = ("It is handled by", "Records attribute it to", "The registry lists", "Official filings name")
_TAIL = (
    "The surrounding documentation covers procurement cycles and archival policies.",
    "Adjacent records describe staffing rosters and equipment manifests.",
    "Related filings track inspection outcomes and renewal deadlines.",
    "Supplementary notes cover logistics corridors and transfer schedules.",
)


def qa_rows(n: int, seed: int = 0) -> list[dict[str, str]]:
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        shape = _SHAPES[int(rng.integers(len(_SHAPES)))]
        adj = _ADJ[int(rng.integers(len(_ADJ)))]
        tag = f"{i:04d}"
        q = shape.format(a=adj, b="ledger" + tag, c="sector" + tag, d="basin" + tag, e="cohort" + tag)
        lead = _LEAD[int(rng.integers(len(_LEAD)))]
        tail = _TAIL[int(rng.integers(len(_TAIL)))]
        ctx = f"The ledger{tag} file for sector{tag} in basin{tag} covers cohort{tag}. {lead} unit{tag}. {tail}"
        out.append({"question": q, "answer": "unit" + tag, "context": ctx})
    return out


def corpus_of(rows: Sequence[dict], source: str = "qa-dataset") -> list[dict]:
    return [{"id": f"{source}-{i:05d}", "text": r["context"], "source": source, "answer": r["answer"]}
            for i, r in enumerate(rows)]


_STOP = frozenset(("a an the of in on at to for by with and or is are was were does do did what which who whom "
                   "whose when where why how about").split())


def mutate(text: str, rng: np.random.Generator) -> str:
    """One light edit (adjacent swap / stop-word drop / terminal punctuation toggle)."""
    words = text.split()
    swaps = [j for j in range(len(words) - 1) if words[j] != words[j + 1]]
    drops = [j for j, w in enumerate(words) if w.lower().strip(".,!?;:") in _STOP]
    kinds = (["swap"] if swaps else []) + (["drop"] if drops and len(words) >= 4 else []) + ["punct"]
    kind = kinds[int(rng.integers(len(kinds)))]
    if kind == "swap":
        j = swaps[int(rng.integers(len(swaps)))]
        words[j], words[j + 1] = words[j + 1], words[j]
        return " ".join(words)
    if kind == "drop":
        j = drops[int(rng.integers(len(drops)))]
        return " ".join(w for k, w in enumerate(words) if k != j)
    return text[:-1] if text[-1] in ".?!" else text + "?"


def linear(i: int, n: int) -> float:
    return i / (n - 1) if n > 1 else 0.0


@dataclasses.dataclass
class Session:
    session_id: str
    questions: Sequence[str]
    n: int
    ramp: Callable[[int, int], float] = linear
    split: float = 0.5
    index: int = 0
    past: list = dataclasses.field(default_factory=list)
    unused: list = dataclasses.field(default_factory=list)

    def __post_init__(self):
        self.unused = list(range(len(self.questions)))

    def draw(self, rng: np.random.Generator) -> tuple[str, str]:
        """(text, origin) of the next query; advances the session."""
        p = self.ramp(self.index, self.n)
        if self.past and float(rng.random()) < p:
            src = self.past[int(rng.integers(len(self.past)))]
            if float(rng.random()) < self.split:
                text, origin = src, "exact_replay"
            else:
                text, origin = mutate(src, rng), "perturbed_replay"
        else:
            if not self.unused:
                raise RuntimeError(f"question pool exhausted after {self.index} queries")
            k = int(rng.integers(len(self.unused)))
            self.unused[k], self.unused[-1] = self.unused[-1], self.unused[k]
            text, origin = self.questions[self.unused.pop()], "fresh"
        self.past.append(text)
        self.index += 1
        return text, origin


_BASE = {1: 0.0, 2: 9.4e-4, 3: 0.25703, 4: 0.53866, 5: 0.53866}  # GPU-s/query by LayerTag value


class LatencyDraws:
    """base(layer) * lognormal(0, sigma), one draw per served query (even base 0)."""

    def __init__(self, sigma: float = 0.25, seed=None):
        self.sigma = sigma
        self.rng = np.random.default_rng(seed)

    def reseed(self, seed) -> None:
        self.rng = np.random.default_rng(seed)

    def sample(self, layer) -> float:
        return _BASE[int(layer)] * float(self.rng.lognormal(mean=0.0, sigma=self.sigma))

    _BASES = np.array([0.0] + [_BASE[i] for i in range(1, 6)])

    def sample_many(self, layers) -> np.ndarray:
        """One draw per entry, in order; a size-n lognormal draw consumes the
        generator exactly like n scalar draws (checked in tests)."""
        layers = np.asarray(layers, dtype=np.int64)
        return self._BASES[layers] * self.rng.lognormal(mean=0.0, sigma=self.sigma, size=layers.size)


def session_stream(questions, n_queries: int, seed: int, s: int, split: float = 0.5):
    """All (text, origin) of session s (texts never depend on routing outcomes)."""
    rng = np.random.default_rng([seed, s, 0])
    sess = Session(f"session_{s:02d}", questions, n_queries, split=split)
    return sess.session_id, [sess.draw(rng) for _ in range(n_queries)]


def simulate_batched(router, questions, *, n_sessions: int, n_queries: int, seed: int, batch: int = 4096,
                     sigma: float = 0.25, vectors_for=None):
    """run_simulation with route_batch; returns per-session lists of JSONL lines
    (the reference's SessionLog.to_jsonl_lines format)."""
    from paper_2506_21593_b200 import validate_query

    if router.latency_model is None:
        router.latency_model = LatencyDraws(sigma)
    logs = []
    for s in range(n_sessions):
        router.reset_session()
        router.latency_model.reseed([seed, s, 1])
        sid, stream = session_stream(questions, n_queries, seed, s)
        qs = [validate_query(t, sid, query_id=f"{sid}-q{i:05d}", issued_at_ns=0) for i, (t, _) in enumerate(stream)]
        V = vectors_for(qs) if vectors_for else None
        res = router.route_batch(qs, vectors=V, span=batch)  # one call: spans pipelined (cascade.py)
        clock, lines = 0, []
        for (ans, ev), (_, origin) in zip(res, stream):
            ev = dataclasses.replace(ev, timestamp_ns=clock)
            clock += int(round(ans.latency_seconds * 1e9))
            rec = ev.to_dict()
            rec["origin"] = origin
            lines.append(json.dumps(rec, ensure_ascii=False))
        logs.append(lines)
    return logs
