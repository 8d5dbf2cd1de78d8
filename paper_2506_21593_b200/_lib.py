"""ctypes binding of libpentarag.so (include/pentarag.h).

The product path has no CPU fallback: if the shared object is missing or the
device is not an sm_100 part, every store constructor raises.  torch is used
only for device memory and the current CUDA stream.
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# PR_LIB overrides the in-tree library (measurement builds only)
LIB_PATH = os.environ.get("PR_LIB") or os.path.join(_HERE, "libpentarag.so")

_lib = None
_lock = threading.Lock()

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_u32 = ctypes.c_uint32
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p

PR_SEARCH_AUTO = 0
PR_SEARCH_EXACT = 1
PR_SEARCH_TENSOR = 2
PR_SEARCH_TENSOR_I8 = 3

PR_OK = 0
PR_ERR_BAD_ARG = -1
PR_ERR_INVALID_VECTOR = -2
PR_ERR_EMPTY = -3
PR_ERR_CUDA = -4
PR_ERR_NOMEM = -5
PR_ERR_UNSUPPORTED = -6


class SearchStats(ctypes.Structure):
    _fields_ = [
        ("queries", c_i64),
        ("tensor_queries", c_i64),
        ("fallback", c_i64),
        ("candidates", c_i64),
        ("nsplit", ctypes.c_int32),
        ("path", ctypes.c_int32),
        ("collected", c_i64),
        ("appended", c_i64),
    ]


ABI_VERSION = 2  # pr_abi_version() of the library these signatures describe
# name -> (restype, argtypes); the exported surface of include/pentarag.h
SIGNATURES = {
    "pr_last_error": (ctypes.c_char_p, []),
    "pr_abi_version": (c_int, []),
    "pr_device_info": (c_int, [c_vp, c_vp, c_vp]),
    "pr_check_unit": (c_int, [c_vp, c_i64, c_int, c_dbl, c_vp, c_vp]),
    "pr_index_create": (c_int, [c_int, c_i64, c_u32, c_vp]),
    "pr_index_destroy": (c_int, [c_vp]),
    "pr_index_count": (c_i64, [c_vp]),
    "pr_index_dim": (c_int, [c_vp]),
    "pr_index_reserve": (c_int, [c_vp, c_i64, c_vp]),
    "pr_index_append": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "pr_index_update_rows": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pr_index_clear": (c_int, [c_vp]),
    "pr_index_truncate": (c_int, [c_vp, c_i64]),
    "pr_index_read_rows": (c_int, [c_vp, c_i64, c_i64, c_vp, c_vp]),
    "pr_index_append_from": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pr_index_search": (c_int, [c_vp, c_vp, c_i64, c_int, c_u32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_index_search_ex": (c_int, [c_vp, c_vp, c_i64, c_int, c_u32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_index_search_floor": (c_int, [c_vp, c_vp, c_i64, c_int, c_u32, c_vp, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_index_search_list": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_u32, c_vp, c_vp, c_vp, c_vp,
                                     c_vp, c_vp]),
    "pr_cascade_gate": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_dbl, c_vp, c_int, c_int, c_int, c_vp, c_vp, c_vp,
                                c_vp, c_vp, c_vp]),
    "pr_recall_gate": (c_int, [c_i64, c_vp, c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp]),
    "pr_cascade_mark_init": (c_int, [c_vp, c_i64, c_vp]),
    "pr_cascade_seeds": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "pr_index_last_stats": (c_int, [c_vp, ctypes.POINTER(SearchStats)]),
    "pr_index_set_timing": (c_int, [c_vp, c_int]),
    "pr_index_scan_time": (c_int, [c_vp, ctypes.POINTER(c_dbl), ctypes.POINTER(c_i64)]),
    "pr_launch_count": (ctypes.c_longlong, []),
    "pr_index_gather_rows": (c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "pr_merge_shards": (c_int, [c_vp, c_vp, c_vp, c_vp, c_int, c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_index_snap_flags": (c_int, [c_vp, c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "pr_kv_create": (c_int, [c_i64, c_vp]),
    "pr_kv_create_ex": (c_int, [c_i64, c_u32, c_vp]),
    "pr_kv_destroy": (c_int, [c_vp]),
    "pr_fingerprint": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "pr_fingerprint_host": (None, [c_vp, c_i64, c_vp]),
    "pr_kv_owner": (c_int, [c_vp, c_vp, c_i64, c_int, c_vp, c_vp]),
    "pr_kv_put_text": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "pr_kv_put_text_owned": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_int, c_int, c_vp]),
    "pr_kv_get_text": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "pr_kv_get_text_owned": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_vp, c_vp]),
    "pr_kv_erase_text": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pr_kv_clear": (c_int, [c_vp, c_vp]),
    "pr_kv_size": (c_i64, [c_vp, c_vp]),
    "pr_kv_capacity": (c_i64, [c_vp]),
    "pr_kv_memory": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_kv_export": (c_i64, [c_vp, c_vp, c_i64, c_vp]),
    "pr_kv_remap": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "pr_l2_fetch_granularity": (c_int, [c_int, c_vp]),
    "pr_hash_embed": (c_int, [c_vp, c_vp, c_i64, c_int, ctypes.c_uint64, c_vp, c_vp, c_vp]),
    "pr_blake2b64_host": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_char_p, c_vp, c_i64]),
    "pr_cascade_route_scratch": (c_i64, [c_i64, c_int, c_i64]),
    "pr_cascade_route": (c_int, [c_vp, c_vp, c_i64, c_vp]),
}


class CascadeSpan(ctypes.Structure):
    """pr_cascade_span (include/pentarag.h): one span of the on-device cascade."""

    _fields_ = [
        ("B", c_i64), ("d_vec", c_vp), ("mode", c_u32),
        ("kv", c_vp), ("d_text", c_vp), ("d_text_off", c_vp), ("d_rep", c_vp),
        ("d_l3_hit", c_vp), ("d_l3_val", c_vp),
        ("sc", c_vp), ("d_sc_limit", c_vp), ("sc_threshold", c_dbl),
        ("l1_blocks", c_int), ("l2_blocks", c_int), ("l3_blocks", c_int),
        ("kb", c_vp), ("seed_k", c_int), ("nlist_hint", c_i64),
        ("d_kb_rows", c_vp), ("d_kb_raw", c_vp), ("d_kb_rep", c_vp), ("d_kb_cnt", c_vp), ("d_nlist", c_vp),
        ("d_slot", c_vp),
        ("probe_l4", c_int), ("akm", c_vp), ("akm_rows", c_i64), ("akm_threshold", c_dbl),
        ("guard", c_vp), ("d_mark", c_vp),
        ("d_prev_rows", c_vp), ("d_prev_cnt", c_vp), ("d_prev_n", c_vp), ("prev_B", c_i64),
        ("d_packed", c_vp),
    ]


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes handle.  Raises if the library is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise errors.NativeLibraryMissing(
                f"{path} is missing: run `python -m paper_2506_21593_b200.build` (there is no CPU fallback)"
            )
        L = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.pr_abi_version() != ABI_VERSION:
            raise errors.NativeLibraryMissing(
                f"{path} has ABI {L.pr_abi_version()}, this package binds ABI {ABI_VERSION}: rebuild it "
                "(`python -m paper_2506_21593_b200.build`)")
        _lib = L
    return _lib


_device_checked = False


def require_device():
    """Fail loudly unless a CUDA device of compute capability 10.0 is present."""
    global _device_checked
    if _device_checked:
        return
    import torch

    if not torch.cuda.is_available():
        raise errors.DeviceUnavailable("paper_2506_21593_b200 needs a CUDA device (sm_100a); none is visible")
    L = load()
    sms, major, minor = c_int(), c_int(), c_int()
    rc = L.pr_device_info(ctypes.byref(sms), ctypes.byref(major), ctypes.byref(minor))
    check(rc)
    _device_checked = True


def last_error() -> str:
    L = load()
    msg = L.pr_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, what: str = ""):
    """Map a C status onto the reference exception taxonomy (errors.py:10-130)."""
    if rc == PR_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == PR_ERR_BAD_ARG:
        raise ValueError(msg)
    if rc == PR_ERR_INVALID_VECTOR:
        raise errors.InvalidVector(msg)
    if rc == PR_ERR_EMPTY:
        raise errors.EmptyKnowledgeBase(msg)
    if rc == PR_ERR_NOMEM:
        raise MemoryError(msg)
    if rc == PR_ERR_UNSUPPORTED:
        raise errors.DeviceUnavailable(msg)
    raise errors.DeviceError(msg)


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def h2d(x, dtype=None):
    """Host array / CPU tensor -> device tensor WITHOUT blocking the host on queued device
    work: staged through the process-wide pinned ring (pinned.py) and copied on the
    current stream.  A pageable source makes the copy synchronous, which stalls a
    pipelined route_batch behind the next span's knowledge-base scan; a fresh pinned
    allocation per call costs milliseconds.  Device tensors pass through."""
    import numpy as np
    import torch

    from . import pinned

    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            return x if dtype is None or x.dtype == dtype else x.to(dtype)
        x = x.numpy()
    a = np.asarray(x)
    if dtype is not None:
        a = a.astype(pinned._NUMPY_OF[dtype], copy=False)
    r = pinned.ring()
    if a.nbytes <= r.cap // 8:
        return r.h2d(a)
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to("cuda", non_blocking=True)
