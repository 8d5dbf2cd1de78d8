"""Exception taxonomy of the drop-in surface.

Same class names, hierarchy and wire ``code`` strings as the reference
(``ragcascade/errors.py:10-130``) for every error the hot path can raise, so a
caller written against the reference catches the same things.  Two additions
are specific to the device build: ``DeviceUnavailable`` (no sm_100 GPU — there
is deliberately no CPU fallback) and ``NativeLibraryMissing``.
"""
from __future__ import annotations


class CascadeError(Exception):
    code = "cascade_error"


class EmptyQuery(CascadeError):
    code = "empty_query"


class EmptyInput(CascadeError):
    code = "empty_input"


class DimensionMismatch(CascadeError):
    code = "dimension_mismatch"


class InvalidVector(CascadeError):
    code = "invalid_vector"


class CorruptSnapshot(CascadeError):
    code = "corrupt_snapshot"


class EmptyKnowledgeBase(CascadeError):
    code = "empty_knowledge_base"


class BackendUnavailable(CascadeError):
    code = "backend_unavailable"


class EmptyContext(CascadeError):
    code = "empty_context"


class AllLayersMissed(CascadeError):
    """No enabled layer answered; carries the trace event (router.py:309-323)."""

    code = "all_layers_missed"

    def __init__(self, message: str, trace_event=None):
        super().__init__(message)
        self.trace_event = trace_event


class DeviceError(CascadeError):
    """A CUDA call inside libpentarag failed."""

    code = "device_error"


class DeviceUnavailable(DeviceError):
    """No usable sm_100a device (the hot path never falls back to the CPU)."""

    code = "device_unavailable"


class NativeLibraryMissing(DeviceUnavailable):
    code = "native_library_missing"


class MalformedJsonl(CascadeError):
    code = "malformed_jsonl"

    def __init__(self, message: str, line_number: int | None = None):
        super().__init__(message)
        self.line_number = line_number
