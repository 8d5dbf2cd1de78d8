"""Service micro-batching.

The reference's ``POST /query`` handler routes each request on its own
(``router.route(q)``, src/service.py:95-100; concurrent requests serialise on
the stores' locks).  ``MicroBatcher`` is the drop-in for that call: request
threads hand their query over and block, one worker coalesces whatever is
waiting (up to ``max_batch``, lingering at most ``max_wait_s`` for more) into
one ``route_batch`` call.  ``route_batch`` is sequential-equivalent, so every
request gets exactly what ``router.route`` would have returned had the
requests been routed one at a time in the order the worker took them
(``served_order`` records it) — including per-request errors such as
AllLayersMissed, which are re-raised in the requesting thread.

    batcher = MicroBatcher(router)
    answer, event = batcher.route(validate_query(text, session_id))   # was: router.route(q)
"""
from __future__ import annotations

import threading
import time
from collections import deque
from concurrent.futures import Future
from typing import Callable

from .errors import CascadeError


class MicroBatcher:
    def __init__(self, router, *, max_batch: int = 4096, max_wait_s: float = 0.0005,
                 batch_fn: Callable | None = None, record_order: bool = False):
        if max_batch < 1:
            raise ValueError("max_batch must be >= 1")
        self.router = router
        self.max_batch = max_batch
        self.max_wait_s = max_wait_s
        self._batch_fn = batch_fn or self._route_batch
        self._pending: deque = deque()
        self._cv = threading.Condition()
        self._closed = False
        self.batches = 0
        self.routed = 0
        self.served_order: list | None = [] if record_order else None
        self._worker = threading.Thread(target=self._run, name="pentarag-microbatcher", daemon=True)
        self._worker.start()

    # -- request side ---------------------------------------------------------
    def submit(self, query) -> Future:
        """Queue one query; the future resolves to (AnswerRecord, RouteTraceEvent)
        or to the CascadeError ``router.route`` would have raised."""
        fut: Future = Future()
        with self._cv:
            if self._closed:
                raise RuntimeError("MicroBatcher is closed")
            self._pending.append((query, fut))
            self._cv.notify()
        return fut

    def route(self, query, timeout: float | None = None):
        """Blocking drop-in for ``router.route(query)``."""
        return self.submit(query).result(timeout)

    def close(self, timeout: float | None = None) -> None:
        """Serve everything already queued, then stop the worker."""
        with self._cv:
            self._closed = True
            self._cv.notify()
        self._worker.join(timeout)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- worker ---------------------------------------------------------------
    def _route_batch(self, queries):
        return self.router.route_batch(queries, capture_errors=True)

    def _take(self):
        with self._cv:
            while not self._pending and not self._closed:
                self._cv.wait()
            if not self._pending:
                return None
            # linger briefly so concurrent requests share the batch
            deadline = time.monotonic() + self.max_wait_s
            while len(self._pending) < self.max_batch and not self._closed:
                left = deadline - time.monotonic()
                if left <= 0:
                    break
                self._cv.wait(left)
            n = min(self.max_batch, len(self._pending))
            return [self._pending.popleft() for _ in range(n)]

    def _run(self) -> None:
        while True:
            batch = self._take()
            if batch is None:
                return
            queries = [q for q, _ in batch]
            try:
                results = self._batch_fn(queries)
            except BaseException as exc:  # noqa: BLE001 - delivered to every waiter of the batch
                for _, fut in batch:
                    fut.set_exception(exc)
                continue
            self.batches += 1
            self.routed += len(batch)
            if self.served_order is not None:
                self.served_order.extend(queries)
            for (_, fut), res in zip(batch, results):
                if isinstance(res, CascadeError):
                    fut.set_exception(res)
                else:
                    fut.set_result(res)
