"""Shared fixtures.  GPU tests are marked ``gpu`` and call the product path
(libpentarag.so through the package); the oracle under ``oracle/`` is only
ever the checker."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100a GPU and libpentarag.so")


def random_unit_vectors(rng: np.random.Generator, n: int, dim: int) -> np.ndarray:
    """Same construction as the reference fixtures (tests/conftest.py:43-46)."""
    raw = rng.normal(size=(n, dim))
    return (raw / np.linalg.norm(raw, axis=1, keepdims=True)).astype(np.float32)


@pytest.fixture()
def rng() -> np.random.Generator:
    return np.random.default_rng(20240817)


def have_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


@pytest.fixture(scope="session", autouse=False)
def gpu():
    if not have_gpu():
        pytest.skip("no CUDA device")
    from paper_2506_21593_b200 import build

    build.build()
    return True
