"""Readers for the committed golden vectors (tests/golden/*.npz, produced by
the reference implementation through tests/golden/make_golden.py)."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import scipy.sparse as sp

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def csr(g: dict, prefix: str) -> sp.csr_matrix:
    shape = tuple(int(v) for v in g[prefix + "_shape"])
    return sp.csr_matrix((g[prefix + "_data"], g[prefix + "_indices"], g[prefix + "_indptr"]), shape=shape)


def steady_case(name: str) -> dict:
    """Golden steady-problem case as plain SciPy/NumPy objects."""
    g = load(name)
    n_t = int(g["n_terms"])
    n_h_terms = len([k for k in g if k.startswith("H") and k.endswith("_shape")])
    case = dict(g)
    case["mass"] = csr(g, "M")
    case["stiffness"] = [csr(g, f"A{t}") for t in range(n_t)]
    case["couplings"] = [csr(g, f"H{t}") for t in range(n_h_terms)]
    case["n_t"] = n_t
    case["boundaries"] = tuple(int(b) for b in g["boundaries"])
    return case
