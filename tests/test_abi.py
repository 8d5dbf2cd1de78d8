"""libpentarag.so loads and exports exactly what include/pentarag.h declares (CPU only).

No compute calls here — only host-side entry points that never touch CUDA.
"""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2506_21593_b200 import _lib, build

    build.build()
    return _lib.load()


def declared_symbols() -> set[str]:
    with open(os.path.join(ROOT, "include", "pentarag.h")) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(pr_[a-z0-9_]+)\s*\(", text))


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, f"declared in pentarag.h but not exported: {missing}"


def test_python_binding_covers_header():
    from paper_2506_21593_b200 import _lib

    assert declared_symbols() == set(_lib.SIGNATURES)


def test_abi_version(lib):
    assert lib.pr_abi_version() == 2


def _fp(lib, b: bytes):
    out = (ctypes.c_uint64 * 2)()
    buf = ctypes.create_string_buffer(b, max(1, len(b)))
    lib.pr_fingerprint_host(ctypes.cast(buf, ctypes.c_void_p), len(b), out)
    return out[0], out[1]


def test_fingerprint_is_byte_exact_and_never_reserved(lib):
    # caches.py:57-58 + tests/test_caches.py:36-45: any byte difference is a new key
    keys = [b"", b"Q1", b"q1", b"Who wrote Hamlet?", b"Who wrote Hamlet? ", b"a" * 15, b"a" * 16, b"a" * 17,
            "ünïcödé".encode(), b"\x00", b"\x00\x00"]
    fps = [_fp(lib, k) for k in keys]
    assert len(set(fps)) == len(keys)
    for tag, hb in fps:
        assert tag >> 31 == 1 and tag < (1 << 32)  # top bit set: never EMPTY (0) or TOMBSTONE (1)
        assert hb < (1 << 32)
    assert _fp(lib, b"Q1") == _fp(lib, b"Q1")


def test_fingerprint_regression_value(lib):
    # pins the hash so host and device (tests/test_gpu_kv.py) and stored tables agree over time
    assert _fp(lib, b"abc") == (2418048503, 3132096303)
    assert _fp(lib, b"query-000000001") == (3201114788, 4107767217)


@pytest.mark.parametrize("token", ["a", "Who", "ledger0007", "_", "9", "x" * 124, "y" * 125, "z" * 300, ""])
@pytest.mark.parametrize("prefix", [b"tok:", b"raw:"])
def test_blake2b_twin_matches_hashlib(lib, token, prefix):
    """The device embedder's keyed BLAKE2b (host twin) == hashlib (embedding.py:131)."""
    import hashlib

    seed = 0x5EED_1024_CA5C_ADE5
    b = token.encode()
    buf = ctypes.create_string_buffer(b, max(1, len(b)))
    got = lib.pr_blake2b64_host(seed, prefix, ctypes.cast(buf, ctypes.c_void_p), len(b))
    want = int.from_bytes(hashlib.blake2b(prefix + b, digest_size=8, key=seed.to_bytes(8, "big")).digest(), "big")
    assert got == want


def test_product_path_refuses_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2506_21593_b200 import DeviceUnavailable, FlatIndex

    with pytest.raises(DeviceUnavailable):
        FlatIndex(dim=8)


def test_search_stats_layout_matches_header():
    """ctypes SearchStats mirrors pr_search_stats field by field (names, order, widths)."""
    from paper_2506_21593_b200 import _lib

    with open(os.path.join(ROOT, "include", "pentarag.h")) as fh:
        text = fh.read()
    body = re.search(r"typedef struct pr_search_stats \{(.*?)\} pr_search_stats;", text, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"(int64_t|int32_t)\s+(\w+);", body)
    width = {"int64_t": ctypes.c_int64, "int32_t": ctypes.c_int32}
    assert [(n, width[t]) for t, n in fields] == list(_lib.SearchStats._fields_)


def test_search_modes_match_header():
    from paper_2506_21593_b200 import _lib

    with open(os.path.join(ROOT, "include", "pentarag.h")) as fh:
        text = fh.read()
    modes = dict((m, int(v)) for m, v in re.findall(r"#define (PR_SEARCH_\w+) (\d+)", text))
    assert modes == {k: getattr(_lib, k) for k in modes}
    assert set(modes) == {"PR_SEARCH_AUTO", "PR_SEARCH_EXACT", "PR_SEARCH_TENSOR", "PR_SEARCH_TENSOR_I8"}


def test_cascade_span_layout_matches_header(tmp_path):
    """ctypes CascadeSpan has pr_cascade_span's size and field offsets (gcc on the header)."""
    import subprocess

    from paper_2506_21593_b200 import _lib

    names = [n for n, _ in _lib.CascadeSpan._fields_]
    src = tmp_path / "off.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "pentarag.h"\nint main(void){\n'
                   '  printf("%zu\\n", sizeof(pr_cascade_span));\n'
                   + "".join(f'  printf("%zu\\n", offsetof(pr_cascade_span, {n}));\n' for n in names) + "  return 0;\n}\n")
    exe = tmp_path / "off"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_lib.CascadeSpan)] + [getattr(_lib.CascadeSpan, n).offset for n in names]
    assert got == want
