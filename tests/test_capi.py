"""The C ABI library builds, loads without a GPU, and exports every symbol
include/sgkkt_b200.h declares; the device path refuses to run without a
GPU instead of falling back to the CPU (CPU only)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "sgkkt_b200.h").read_text()
    return sorted(set(re.findall(r"\b(sgk_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_2512_23804_b200 import _lib

    handle = _lib.load_without_device()
    names = _declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(handle, name), f"{name} declared in the header but not exported"
    assert set(_lib.EXPORTED) <= set(names) | {"sgk_last_error", "sgk_version", "sgk_launch_count"}


def test_so_is_sm100a_only():
    import subprocess

    lib = ROOT / "paper_2512_23804_b200" / "libsgkkt_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_argument_validation_without_gpu():
    from paper_2512_23804_b200 import _lib

    h = _lib.load_without_device()
    assert h.sgk_version() == 1
    # validation happens before any device work
    assert h.sgk_program_apply(None, None, 0, None, 1, None, None, None, None, 256, None) == -1
    assert b"null" in h.sgk_last_error()
    assert h.sgk_trisolve(None, None, None, None, None, None, None, 1, 1, None) == -1


def test_no_cpu_fallback(monkeypatch):
    import torch

    from paper_2512_23804_b200 import _lib

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError, match="CUDA device"):
        _lib.lib()
    import numpy as np

    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply
    import scipy.sparse as sp

    op = KroneckerSumOperator(couplings=[sp.identity(2, format="csr")], operators=[sp.identity(3, format="csr")])
    with pytest.raises(RuntimeError):
        kron_apply(op, np.zeros((3, 2)))
