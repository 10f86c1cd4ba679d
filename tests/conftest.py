"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and run on the B200
(`pytest -m gpu`); everything else runs on the CPU build container."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

SEED = 20240817  # reference test seed (reference tests/conftest.py:18-20)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsgkkt_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container (run with -m gpu on the B200)")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """A fresh checkout has no libsgkkt_b200.so (git-ignored): build it once
    (nvcc cross-compiles without a GPU) so the ABI tests see the real file."""
    from paper_2512_23804_b200 import _lib

    if not _lib.library_path().exists():
        import __graft_entry__

        __graft_entry__.build()
    yield


@pytest.fixture
def rng():
    return np.random.default_rng(SEED)
