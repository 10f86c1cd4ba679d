"""B200-native hot path of the stochastic Galerkin KKT solver of arXiv
2512.23804 (reference package `sgkkt`): the Galerkin matvec
W = sum_t A_t V H_t^T, the hGS / hGSoc preconditioners built on it, and the
CG / MINRES / FGMRES drivers — hand-written sm_100a CUDA behind the C ABI in
include/sgkkt_b200.h, with the reference's Python call signatures.

Host-only modules (setup: basis, fem, random_field, problems, program) import
without a GPU; the device modules raise RuntimeError on use when
libsgkkt_b200.so or a CUDA device is missing (no CPU fallback).
"""

from __future__ import annotations

import importlib

__version__ = "0.1.0"

_SUBMODULES = (
    "basis",
    "fem",
    "random_field",
    "problems",
    "program",
    "operators",
    "linalg",
    "preconditioners",
    "krylov",
    "timedep",
    "vec",
    "device",
)


def __getattr__(name):
    if name in _SUBMODULES:
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
