"""Host-side problem assembly for the five BASELINE.json configurations
(setup only; mirrors `sgkkt.problems`, reference pkg/src/sgkkt/problems.py:91-177,
re-composed for the BASELINE settings: unit square, Legendre chaos for the
affine configs, separable KL, the forward problem -div(a grad u) = 1, the
sin target).

    cfg1  forward,  n=32,  affine Legendre, m=4,  p=3  (n_xi=35,  n_t=5)   sigma=0.2 ell=0.5
    cfg2  control,  n=64,  affine Legendre, m=6,  p=3  (n_xi=84,  n_t=7)   sigma=0.3 beta=1e-2
    cfg3  forward,  n=64,  lognormal Hermite, m=6, p=3, coefficient degree 6 (n_t=924), sigma_g=0.5 ell=1
    cfg4  matvec,   n=256, affine Legendre, m=10, p=4  (n_xi=1001, n_t=11)
    cfg5  control,  n=128, affine Legendre, m=8,  p=4  (n_xi=495, n_t=9)   sigma=0.3 beta in {1e-2,1e-4,1e-6}

Unspecified by BASELINE.json and chosen here: correlation length
1.0 for cfgs 2, 4, 5 (the reference default), sigma=0.3 for cfg4, mean 1,
gamma = 1 (reference default).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import fem
from .basis import (
    LevelPartition,
    MultiIndexSet,
    TripleProductSet,
    build_triple_products,
    enumerate_multi_indices,
    level_partition,
)
from .random_field import CovarianceSpec, GpcCoefficientField, KLModes, affine_coefficient, kl_expand, lognormal_coefficient

__all__ = ["BASELINE_CONFIGS", "ProblemBundle", "build_problem", "sin_target"]


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    kind: str  # "forward" | "control" | "matvec"
    n: int
    m_xi: int
    p: int
    family: str
    coefficient: str  # "affine" | "lognormal"
    sigma: float
    ell: float
    coefficient_degree: int = 1
    beta: float = 1e-2
    gamma: float = 1.0
    lo: float = 0.0
    hi: float = 1.0


BASELINE_CONFIGS = {
    1: ConfigSpec("cfg1", "forward", 32, 4, 3, "legendre", "affine", 0.2, 0.5),
    2: ConfigSpec("cfg2", "control", 64, 6, 3, "legendre", "affine", 0.3, 1.0, beta=1e-2),
    3: ConfigSpec("cfg3", "forward", 64, 6, 3, "hermite", "lognormal", 0.5, 1.0, coefficient_degree=6),
    4: ConfigSpec("cfg4", "matvec", 256, 10, 4, "legendre", "affine", 0.3, 1.0),
    5: ConfigSpec("cfg5", "control", 128, 8, 4, "legendre", "affine", 0.3, 1.0, beta=1e-2),
}


def sin_target(x, y):
    return np.sin(np.pi * x) * np.sin(np.pi * y)


@dataclass
class ProblemBundle:
    spec: ConfigSpec
    grid: fem.Grid
    basis: MultiIndexSet
    partition: LevelPartition
    triple: TripleProductSet
    modes: KLModes
    coefficient: GpcCoefficientField
    mass: object
    stiffness: list
    extras: dict = field(default_factory=dict)

    @property
    def n_h(self) -> int:
        return self.grid.n_interior

    @property
    def n_xi(self) -> int:
        return self.basis.size

    @property
    def n_terms(self) -> int:
        return len(self.stiffness)

    def forward_rhs(self) -> np.ndarray:
        """b = f (x) e_0 for -div(a grad u) = 1 (E[psi_0] = 1, E[psi_k] = 0)."""
        b = np.zeros((self.n_h, self.n_xi))
        b[:, 0] = fem.load_vector(self.grid, 1.0)
        return b

    def target(self) -> np.ndarray:
        t = np.zeros((self.n_h, self.n_xi))
        t[:, 0] = fem.interpolate_nodal(self.grid, sin_target)
        return t


def build_problem(cfg: int | ConfigSpec, *, n: int | None = None, kl_method: str = "separable",
                  beta: float | None = None) -> ProblemBundle:
    spec = BASELINE_CONFIGS[cfg] if isinstance(cfg, int) else cfg
    if n is not None or beta is not None:
        from dataclasses import replace

        spec = replace(spec, n=n if n is not None else spec.n, beta=beta if beta is not None else spec.beta)
    grid = fem.build_grid(spec.n, spec.lo, spec.hi)
    basis = enumerate_multi_indices(spec.m_xi, spec.p)
    partition = level_partition(basis)
    modes = kl_expand(CovarianceSpec(sigma_k=spec.sigma, ell1=spec.ell, ell2=spec.ell, mean=1.0), grid,
                      spec.m_xi, method=kl_method)
    if spec.coefficient == "affine":
        coeff_idx = enumerate_multi_indices(spec.m_xi, 1)
        gpc = affine_coefficient(modes, spec.family)
    else:
        coeff_idx = enumerate_multi_indices(spec.m_xi, spec.coefficient_degree)
        gpc = lognormal_coefficient(modes, coeff_idx)
    triple = build_triple_products(basis, coeff_idx, spec.gamma, family=spec.family)
    mass = fem.assemble_mass(grid)
    stiffness = [fem.assemble_stiffness(grid, f) for f in gpc.coeff_fields]
    if len(stiffness) != math.comb(spec.m_xi + spec.coefficient_degree, spec.coefficient_degree):
        raise AssertionError("coefficient term count mismatch")
    return ProblemBundle(spec, grid, basis, partition, triple, modes, gpc, mass, stiffness)


def steady_system(bundle: ProblemBundle, beta: float | None = None):
    """SteadyKKT for a control configuration (target in column 0)."""
    from .operators import SteadyKKT

    return SteadyKKT(mass=bundle.mass, stiffness=bundle.stiffness, triple=bundle.triple,
                     beta=bundle.spec.beta if beta is None else beta, gamma=bundle.spec.gamma,
                     target=bundle.target())
