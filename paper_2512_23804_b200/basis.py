"""Host-side chaos combinatorics: multi-indices, triple-product couplings H_t,
degree-level partition.

Setup only (runs once per problem, on the host).  Mirrors the reference
interface `sgkkt.basis` (reference: pkg/src/sgkkt/basis.py):

* ``enumerate_multi_indices``  — basis.py:70-80 (graded; inside a degree the
  tuples are in descending lexicographic order, so the first variable's
  exponent drops first; the zero tuple comes first)
* ``univariate_triple``        — basis.py:83-100 (Hermite closed form), plus
  the Legendre closed form BASELINE.json configs 1,2,4,5 need (normalised
  Legendre polynomials, xi ~ U(-1,1)); the reference has Hermite only.
* ``build_triple_products``    — basis.py:133-175 (exact zeros dropped, no
  threshold; matrices[0] is the identity)
* ``LevelPartition`` / ``level_partition`` — basis.py:178-203
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import scipy.sparse as sp
from scipy.sparse import csr_matrix

__all__ = [
    "FAMILIES",
    "LevelPartition",
    "MultiIndexSet",
    "TripleProductSet",
    "build_triple_products",
    "enumerate_multi_indices",
    "hermite_triple",
    "legendre_triple",
    "level_partition",
    "univariate_triple",
]

FAMILIES = ("hermite", "legendre")


@dataclass(frozen=True)
class MultiIndexSet:
    """Graded total-degree multi-index set (reference basis.py:31-56)."""

    m_xi: int
    p: int
    indices: tuple[tuple[int, ...], ...]

    @property
    def size(self) -> int:
        return len(self.indices)

    def degree_sizes(self) -> list[int]:
        out = [0] * (self.p + 1)
        for idx in self.indices:
            out[sum(idx)] += 1
        return out

    def as_array(self) -> np.ndarray:
        return np.array(self.indices, dtype=np.int64).reshape(self.size, self.m_xi)


def _compositions(total: int, parts: int) -> list[tuple[int, ...]]:
    """All `parts`-tuples of nonnegative ints summing to `total`, in
    descending lexicographic order (stars and bars)."""
    out = []
    for bars in itertools.combinations(range(total + parts - 1), parts - 1):
        prev = -1
        comp = []
        for b in bars:
            comp.append(b - prev - 1)
            prev = b
        comp.append(total + parts - 1 - prev - 1)
        out.append(tuple(comp))
    out.sort(reverse=True)
    return out


def enumerate_multi_indices(m_xi: int, p: int) -> MultiIndexSet:
    if m_xi < 1:
        raise ValueError("need at least one random variable")
    if p < 0:
        raise ValueError("degree must be nonnegative")
    idx: list[tuple[int, ...]] = []
    for d in range(p + 1):
        idx.extend(_compositions(d, m_xi))
    if len(idx) != math.comb(m_xi + p, p):
        raise AssertionError("multi-index count mismatch")
    return MultiIndexSet(m_xi=m_xi, p=p, indices=tuple(idx))


def _triangle_half(i: int, j: int, k: int) -> int | None:
    if i < 0 or j < 0 or k < 0:
        raise ValueError("degrees must be nonnegative")
    tot = i + j + k
    if tot & 1:
        return None
    s = tot // 2
    if i > s or j > s or k > s:
        return None
    return s


def hermite_triple(i: int, j: int, k: int) -> float:
    """E[h_i h_j h_k] for unit-variance probabilists' Hermite polynomials,
    xi ~ N(0,1): sqrt(i! j! k!) / ((s-i)! (s-j)! (s-k)!), s = (i+j+k)/2."""
    s = _triangle_half(i, j, k)
    if s is None:
        return 0.0
    f = math.factorial
    return math.sqrt(f(i) * f(j) * f(k)) / (f(s - i) * f(s - j) * f(s - k))


def legendre_triple(i: int, j: int, k: int) -> float:
    """E[L_i L_j L_k] for Legendre polynomials normalised to unit variance
    under xi ~ U(-1,1): sqrt((2i+1)(2j+1)(2k+1)) * (i j k; 0 0 0)^2 with the
    Wigner 3j closed form (Adams / Neumann formula)."""
    s = _triangle_half(i, j, k)
    if s is None:
        return 0.0
    f = math.factorial
    w2 = (f(2 * s - 2 * i) * f(2 * s - 2 * j) * f(2 * s - 2 * k)) / f(2 * s + 1)
    w2 *= (f(s) / (f(s - i) * f(s - j) * f(s - k))) ** 2
    return math.sqrt((2 * i + 1) * (2 * j + 1) * (2 * k + 1)) * w2


def univariate_triple(i: int, j: int, k: int, family: str = "hermite") -> float:
    if family == "hermite":
        return hermite_triple(i, j, k)
    if family == "legendre":
        return legendre_triple(i, j, k)
    raise ValueError(f"unknown chaos family {family!r}")


@lru_cache(maxsize=64)
def _triple_table(max_c: int, max_b: int, family: str) -> np.ndarray:
    tab = np.empty((max_c + 1, max_b + 1, max_b + 1))
    for a in range(max_c + 1):
        for b in range(max_b + 1):
            for c in range(max_b + 1):
                tab[a, b, c] = univariate_triple(a, b, c, family)
    tab.setflags(write=False)
    return tab


@dataclass(frozen=True)
class TripleProductSet:
    """H_t = E[psi_t psi_j psi_k] over the solution basis for every
    coefficient index t (reference basis.py:103-130)."""

    matrices: list[csr_matrix]
    variance_penalty: csr_matrix
    objective_weight: csr_matrix
    gamma: float
    family: str = "hermite"

    @property
    def n_terms(self) -> int:
        return len(self.matrices)

    @property
    def size(self) -> int:
        return self.matrices[0].shape[0]

    @property
    def weight_diagonal(self) -> np.ndarray:
        return self.objective_weight.diagonal()


def build_triple_products(
    basis: MultiIndexSet,
    coeff_indices: MultiIndexSet,
    gamma: float = 1.0,
    family: str = "hermite",
) -> TripleProductSet:
    if basis.m_xi != coeff_indices.m_xi:
        raise ValueError("basis and coefficient indices use different variable counts")
    if gamma < 0:
        raise ValueError("gamma must be nonnegative")
    if family not in FAMILIES:
        raise ValueError(f"unknown chaos family {family!r}")
    n = basis.size
    b = basis.as_array()
    max_b = int(b.max()) if n else 0
    max_c = max((max(t) for t in coeff_indices.indices), default=0)
    tab = _triple_table(max_c, max_b, family)
    # per-variable factor matrices E[v][deg] = tab[deg, b[:,v], b[:,v]^T]
    mats = []
    for ell in coeff_indices.indices:
        prod = None
        for v, deg in enumerate(ell):
            fac = tab[deg][b[:, v][:, None], b[:, v][None, :]]
            prod = fac.copy() if prod is None else prod * fac
        if prod is None:
            prod = np.ones((n, n))
        rows, cols = np.nonzero(prod)
        h = sp.coo_matrix((prod[rows, cols], (rows, cols)), shape=(n, n)).tocsr()
        h.sum_duplicates()
        h.sort_indices()
        mats.append(h)
    diag_pen = np.ones(n)
    if n:
        diag_pen[0] = 0.0
    pen_idx = np.flatnonzero(diag_pen)
    variance_penalty = sp.coo_matrix(
        (np.ones(pen_idx.size), (pen_idx, pen_idx)), shape=(n, n)
    ).tocsr()
    weight = sp.diags(1.0 + gamma * diag_pen, format="csr")
    return TripleProductSet(
        matrices=mats,
        variance_penalty=variance_penalty,
        objective_weight=weight,
        gamma=float(gamma),
        family=family,
    )


@dataclass(frozen=True)
class LevelPartition:
    """Cumulative column counts closing each degree level."""

    boundaries: tuple[int, ...]

    @property
    def n_levels(self) -> int:
        return len(self.boundaries)

    def ranges(self) -> list[tuple[int, int]]:
        lows = (0,) + tuple(self.boundaries[:-1])
        return list(zip(lows, self.boundaries))


def level_partition(basis: MultiIndexSet) -> LevelPartition:
    bounds = tuple(math.comb(basis.m_xi + d, d) for d in range(basis.p + 1))
    part = LevelPartition(boundaries=bounds)
    if [hi - lo for lo, hi in part.ranges()] != basis.degree_sizes():
        raise AssertionError("level boundaries disagree with the degree sizes")
    return part
