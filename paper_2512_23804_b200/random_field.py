"""Host-side Karhunen–Loève expansion of the separable exponential covariance
and the gPC coefficient fields built from it (setup only).

Mirrors `sgkkt.random_field` (reference pkg/src/sgkkt/random_field.py):
Nyström on the element Gauss points with the uniform weight (h/2)^2
(random_field.py:71-106), sign fixed so the first significant entry of each
mode is positive, affine coefficient = mean then scaled modes
(:120-127), lognormal coefficient = mean * prod_i g_i^k_i / sqrt(k_i!)
(:130-151).

Additions for BASELINE.json:
* ``kl_expand(..., method="separable")`` — the covariance
  sigma^2 exp(-|dx|/l1 - |dy|/l2) is a product of 1-D kernels and the Gauss
  points form a tensor grid, so the weighted Nyström matrix is the
  Kronecker product of two 1-D ones and its eigenpairs are products of 1-D
  eigenpairs (the reference's own test oracle uses the 1-D problem,
  tests/oracles.py:310-322).  The dense (4n^2)^2 eigenproblem of the
  reference is infeasible at n=128/256 (34 GB / 550 GB).
* ``affine_coefficient(..., family="legendre")`` — with xi_k ~ U(-1,1) the
  first normalised Legendre polynomial is sqrt(3) xi, so the gPC coefficient
  of psi_{e_k} is mode_k / sqrt(3) (for Hermite, He_1 = xi, factor 1).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.linalg

from .basis import MultiIndexSet
from .fem import CoefficientField, Grid

__all__ = [
    "CovarianceSpec",
    "GpcCoefficientField",
    "KLModes",
    "affine_coefficient",
    "kl_expand",
    "lognormal_coefficient",
]


@dataclass(frozen=True)
class CovarianceSpec:
    sigma_k: float
    ell1: float = 1.0
    ell2: float = 1.0
    mean: float = 1.0

    def __post_init__(self):
        if self.sigma_k < 0:
            raise ValueError("sigma_k must be nonnegative")
        if self.ell1 <= 0 or self.ell2 <= 0:
            raise ValueError("correlation lengths must be positive")

    def kernel(self, x1, y1, x2, y2) -> np.ndarray:
        return self.sigma_k**2 * np.exp(-np.abs(x1 - x2) / self.ell1 - np.abs(y1 - y2) / self.ell2)


@dataclass(frozen=True)
class KLModes:
    eigenvalues: np.ndarray
    mode_fields: list[CoefficientField]
    mean_field: CoefficientField

    @property
    def m_xi(self) -> int:
        return len(self.mode_fields)


def _fix_sign(kappa: np.ndarray) -> np.ndarray:
    thresh = 1e-12 * max(float(np.abs(kappa).max()), 1.0)
    sig = np.flatnonzero(np.abs(kappa) > thresh)
    if sig.size and kappa[sig[0]] < 0:
        return -kappa
    return kappa


def _modes_from(vals, vecs, grid: Grid, spec: CovarianceSpec, m_xi: int) -> KLModes:
    w = grid.quad_weight
    fields = []
    for i in range(m_xi):
        kappa = _fix_sign(vecs[:, i] / math.sqrt(w))
        fields.append(CoefficientField(values=(math.sqrt(vals[i]) * kappa).reshape(grid.gauss_x.shape)))
    mean = CoefficientField(values=np.full(grid.gauss_x.shape, spec.mean))
    return KLModes(eigenvalues=np.asarray(vals[:m_xi]), mode_fields=fields, mean_field=mean)


def _kl_dense(spec: CovarianceSpec, grid: Grid, m_xi: int) -> KLModes:
    xs = grid.gauss_x.ravel()
    ys = grid.gauss_y.ravel()
    n = xs.size
    sym = grid.quad_weight * spec.kernel(xs[:, None], ys[:, None], xs[None, :], ys[None, :])
    vals, vecs = scipy.linalg.eigh(sym, subset_by_index=[n - m_xi, n - 1])
    order = np.argsort(vals)[::-1]
    return _modes_from(np.maximum(vals[order], 0.0), vecs[:, order], grid, spec, m_xi)


def _kl_separable(spec: CovarianceSpec, grid: Grid, m_xi: int) -> KLModes:
    n = grid.n_cells
    half = grid.h / 2.0
    # 1-D Gauss abscissae in index order 2*e + q (q=0: -g, q=1: +g)
    centers = grid.lo + (np.arange(n) + 0.5) * grid.h
    pts = np.stack([centers - half * GAUSS, centers + half * GAUSS], axis=1).ravel()

    def one_d(ell):
        k = half * np.exp(-np.abs(pts[:, None] - pts[None, :]) / ell)
        lam, vec = np.linalg.eigh(k)
        o = np.argsort(lam)[::-1]
        return np.maximum(lam[o], 0.0), vec[:, o]

    lx, ux = one_d(spec.ell1)
    ly, uy = (lx, ux) if spec.ell2 == spec.ell1 else one_d(spec.ell2)
    cand = min(m_xi, lx.size)
    prod = spec.sigma_k**2 * (lx[:cand, None] * ly[None, :cand])
    a_idx, b_idx = np.unravel_index(np.arange(cand * cand), (cand, cand))
    order = np.lexsort((b_idx, a_idx, -prod.ravel()))[:m_xi]
    # Gauss point (element e=(ex,ey), q=(qx,qy)) -> 1-D indices (2ex+qx, 2ey+qy)
    ey, ex = np.divmod(np.arange(n * n), n)
    qx = np.array([0, 1, 0, 1])
    qy = np.array([0, 0, 1, 1])
    ix = (2 * ex[:, None] + qx[None, :]).ravel()
    iy = (2 * ey[:, None] + qy[None, :]).ravel()
    vals = np.empty(m_xi)
    vecs = np.empty((ix.size, m_xi))
    for col, flat in enumerate(order):
        a, b = a_idx[flat], b_idx[flat]
        vals[col] = prod.ravel()[flat]
        vecs[:, col] = ux[ix, a] * uy[iy, b]
    return _modes_from(vals, vecs, grid, spec, m_xi)


GAUSS = 1.0 / math.sqrt(3.0)


def kl_expand(spec: CovarianceSpec, grid: Grid, m_xi: int, method: str = "auto") -> KLModes:
    npts = grid.gauss_x.size
    if not 1 <= m_xi <= npts:
        raise ValueError(f"m_xi must be in [1, {npts}]")
    if spec.sigma_k == 0.0:
        zeros = [CoefficientField(values=np.zeros(grid.gauss_x.shape)) for _ in range(m_xi)]
        return KLModes(np.zeros(m_xi), zeros, CoefficientField(np.full(grid.gauss_x.shape, spec.mean)))
    if method == "auto":
        method = "dense" if npts <= 4096 else "separable"
    if method == "dense":
        return _kl_dense(spec, grid, m_xi)
    if method == "separable":
        return _kl_separable(spec, grid, m_xi)
    raise ValueError(f"unknown KL method {method!r}")


@dataclass(frozen=True)
class GpcCoefficientField:
    coeff_fields: list[CoefficientField]

    @property
    def n_terms(self) -> int:
        return len(self.coeff_fields)


def affine_coefficient(modes: KLModes, family: str = "hermite") -> GpcCoefficientField:
    scale = {"hermite": 1.0, "legendre": 1.0 / math.sqrt(3.0)}.get(family)
    if scale is None:
        raise ValueError(f"unknown chaos family {family!r}")
    fields = [modes.mean_field] + [CoefficientField(f.values * scale) for f in modes.mode_fields]
    return GpcCoefficientField(coeff_fields=fields)


def lognormal_coefficient(modes: KLModes, coeff_basis: MultiIndexSet) -> GpcCoefficientField:
    if coeff_basis.m_xi != modes.m_xi:
        raise ValueError("coefficient basis and modes use different variable counts")
    mean = modes.mean_field.values
    if np.any(mean <= 0):
        raise ValueError("lognormal mean field must be strictly positive")
    g = [f.values for f in modes.mode_fields]
    out = []
    for idx in coeff_basis.indices:
        c = mean.copy()
        for i, k in enumerate(idx):
            if k:
                c = c * g[i] ** k / math.sqrt(math.factorial(k))
        out.append(CoefficientField(values=c))
    return GpcCoefficientField(coeff_fields=out)
