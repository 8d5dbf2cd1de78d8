"""RCFLATIX snapshots (reference index.py:198-261) against fixtures written by the
real reference (tests/golden/make_golden.py snapshot).

CPU: the host parser (header, crc, sidecar) and the corrupt cases.
GPU: bulk device restore == the reference's per-record restore (ids, payloads,
search hits) and snapshot() bytes identical to the reference's.
"""
from __future__ import annotations

import base64
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "snapshot.json")) as fh:
        return json.load(fh)


def b64(s):
    return base64.b64decode(s)


def test_parser_reads_reference_snapshot(golden):
    from paper_2506_21593_b200.index import parse_snapshot

    dim, vecs, recs = parse_snapshot(b64(golden["snapshot_b64"]))
    assert dim == golden["dim"] and vecs.shape == (30, dim)
    assert [r["id"] for r in recs] == golden["restored_ids"]
    assert [r["payload"] for r in recs] == golden["restored_payloads"]
    assert np.allclose(np.linalg.norm(vecs.astype(np.float64), axis=1), 1.0, atol=1e-5)


@pytest.mark.parametrize("case", ["bad_magic", "bad_version", "bad_crc", "short"])
def test_parser_rejects_corrupt(golden, case):
    from paper_2506_21593_b200 import CorruptSnapshot
    from paper_2506_21593_b200.index import parse_snapshot

    assert golden["bad"][case]["error"] == "CorruptSnapshot"
    with pytest.raises(CorruptSnapshot):
        parse_snapshot(b64(golden["bad"][case]["b64"]))


def _hits(idx, queries, k):
    return [[[h.entry_id, h.score, h.rank] for h in idx.search(np.asarray(q, dtype=np.float32), k)] for q in queries]


@pytest.mark.gpu
def test_device_restore_matches_reference(gpu, golden):
    from paper_2506_21593_b200 import FlatIndex

    snap = b64(golden["snapshot_b64"])
    idx = FlatIndex.restore(snap)
    assert list(idx.entry_ids()) == golden["restored_ids"]
    assert [idx.payload(e) for e in idx.entry_ids()] == golden["restored_payloads"]
    assert _hits(idx, golden["queries"], 5) == golden["hits"]
    assert idx.snapshot() == snap  # byte-identical round trip


@pytest.mark.gpu
def test_device_restore_duplicate_ids_upsert(gpu, golden):
    from paper_2506_21593_b200 import FlatIndex
    from paper_2506_21593_b200.index import parse_snapshot

    blob = b64(golden["dup_b64"])
    idx = FlatIndex.restore(blob)
    assert list(idx.entry_ids()) == golden["dup_ids"]
    assert [idx.payload(e) for e in idx.entry_ids()] == golden["dup_payloads"]
    _, vecs, _ = parse_snapshot(blob)
    assert _hits(idx, vecs[:3], 6) == golden["dup_hits"]
    assert idx.snapshot() == b64(golden["dup_snapshot_b64"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["bad_magic", "bad_version", "bad_crc", "short", "not_unit"])
def test_device_restore_errors(gpu, golden, case):
    from paper_2506_21593_b200 import FlatIndex, errors

    want = getattr(errors, golden["bad"][case]["error"])
    with pytest.raises(want):
        FlatIndex.restore(b64(golden["bad"][case]["b64"]))
