"""Host-side producers (basis, FEM, KL) against the reference's golden
outputs and independent quadrature oracles (CPU only)."""

from __future__ import annotations

import math

import numpy as np
import pytest
import scipy.sparse as sp

from golden_io import csr, load
from paper_2512_23804_b200 import basis, fem, random_field
from paper_2512_23804_b200.problems import BASELINE_CONFIGS, build_problem


@pytest.fixture(scope="module")
def g():
    return load("basis_fem")


def test_multi_indices_match_reference(g):
    assert np.array_equal(basis.enumerate_multi_indices(3, 3).as_array(), g["mi_3_3"])
    assert np.array_equal(basis.enumerate_multi_indices(4, 2).as_array(), g["mi_4_2"])
    assert basis.level_partition(basis.enumerate_multi_indices(3, 3)).boundaries == tuple(g["levels_3_3"])


def test_counts_and_known_answers():
    # reference tests/test_basis.py:15-20, :60-63
    assert basis.enumerate_multi_indices(3, 3).size == 20
    assert basis.enumerate_multi_indices(4, 4).size == 70
    assert basis.enumerate_multi_indices(6, 3).size == 84
    assert basis.univariate_triple(1, 1, 2) == pytest.approx(math.sqrt(2.0), abs=1e-15)
    assert basis.univariate_triple(1, 1, 3) == 0.0
    with pytest.raises(ValueError):
        basis.univariate_triple(-1, 0, 0)
    with pytest.raises(ValueError):
        basis.enumerate_multi_indices(0, 2)


def test_hermite_triples_match_reference(g):
    tab = g["hermite_table"]
    for i in range(5):
        for j in range(5):
            for k in range(5):
                assert basis.hermite_triple(i, j, k) == tab[i, j, k]
    mi = basis.enumerate_multi_indices(3, 3)
    tp = basis.build_triple_products(mi, basis.enumerate_multi_indices(3, 2), gamma=1.0)
    assert len(tp.matrices) == int(g["n_H"])
    for t, h in enumerate(tp.matrices):
        ref = csr(g, f"H{t}")
        assert (h != ref).nnz == 0
        assert np.array_equal(h.indptr, ref.indptr) and np.array_equal(h.indices, ref.indices)


def _gauss_legendre_triple(i, j, k, n=16):
    x, w = np.polynomial.legendre.leggauss(n)
    w = w / 2.0  # uniform density on [-1, 1]
    def p(d):
        c = np.zeros(d + 1)
        c[d] = 1.0
        return np.polynomial.legendre.legval(x, c) * math.sqrt(2 * d + 1)
    return float(np.sum(w * p(i) * p(j) * p(k)))


def test_legendre_triples_match_quadrature():
    # no reference implementation (Hermite only): pinned by Gauss-Legendre
    for i in range(6):
        for j in range(6):
            for k in range(6):
                assert basis.legendre_triple(i, j, k) == pytest.approx(_gauss_legendre_triple(i, j, k), abs=1e-12)
    # orthonormality: E[L_0 L_j L_k] = delta_jk
    for j in range(5):
        assert basis.legendre_triple(0, j, j) == pytest.approx(1.0, abs=1e-14)


def test_triple_products_legendre_structure():
    mi = basis.enumerate_multi_indices(3, 2)
    tp = basis.build_triple_products(mi, basis.enumerate_multi_indices(3, 1), gamma=1.0, family="legendre")
    assert (tp.matrices[0] != sp.identity(mi.size)).nnz == 0
    for h in tp.matrices:
        assert abs(h - h.T).max() == 0.0
    # first-order Hermite and Legendre share the sparsity pattern
    tph = basis.build_triple_products(mi, basis.enumerate_multi_indices(3, 1), gamma=1.0)
    for a, b in zip(tp.matrices, tph.matrices):
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)


def test_fem_matches_reference(g):
    grid = fem.build_grid(5)
    assert np.allclose(grid.gauss_x, g["gauss_x"], atol=1e-15, rtol=0)
    assert np.allclose(grid.gauss_y, g["gauss_y"], atol=1e-15, rtol=0)
    for mine, key in ((fem.assemble_mass(grid), "mass"), (fem.assemble_mass(grid, False), "mass_full")):
        ref = csr(g, key)
        assert np.array_equal(mine.indptr, ref.indptr) and np.array_equal(mine.indices, ref.indices)
        assert np.abs(mine.data - ref.data).max() <= 1e-15
    field = fem.CoefficientField(g["field"])
    st = fem.assemble_stiffness(grid, field)
    ref = csr(g, "stiff")
    assert np.array_equal(st.indptr, ref.indptr) and np.array_equal(st.indices, ref.indices)
    assert np.abs(st.data - ref.data).max() <= 1e-14
    assert np.allclose(fem.interpolate_nodal(grid, lambda x, y: np.sin(x) * np.cos(y)), g["interp"], atol=1e-15)


def test_fem_known_answers_and_unit_square():
    # reference tests/test_fem.py:59-62 (total mass 4 on [-1,1]^2), :81-91 (diag 8/3)
    grid = fem.build_grid(8)
    full = fem.assemble_mass(grid, eliminate_boundary=False)
    assert full.sum() == pytest.approx(4.0, abs=1e-13)
    st = fem.assemble_stiffness(grid, fem.constant_field(grid, 1.0))
    assert np.allclose(st.diagonal(), 8.0 / 3.0, atol=1e-14)
    unit = fem.build_grid(8, 0.0, 1.0)
    assert fem.assemble_mass(unit, eliminate_boundary=False).sum() == pytest.approx(1.0, abs=1e-14)
    # forward-problem load vector: int psi_i = h^2 for interior nodes
    assert np.allclose(fem.load_vector(unit), (1.0 / 8) ** 2, atol=1e-15)
    # stiffness is h-independent in 2-D
    assert abs(fem.assemble_stiffness(unit, fem.constant_field(unit, 1.0)) - st).max() <= 1e-14


def test_all_matrices_share_one_pattern():
    b = build_problem(1)
    for a in b.stiffness + [b.mass]:
        assert np.array_equal(a.indptr, b.mass.indptr) and np.array_equal(a.indices, b.mass.indices)
    n = b.spec.n
    assert b.mass.nnz == (3 * (n - 1) - 2) ** 2


def test_kl_dense_matches_reference(g):
    spec = random_field.CovarianceSpec(sigma_k=0.4, ell1=0.7, ell2=1.3)
    kl = random_field.kl_expand(spec, fem.build_grid(6), 5, method="dense")
    assert np.allclose(kl.eigenvalues, g["kl_vals"], rtol=1e-10, atol=1e-14)
    modes = np.stack([f.values for f in kl.mode_fields])
    assert np.allclose(modes, g["kl_modes"], rtol=1e-8, atol=1e-10)
    logn = random_field.lognormal_coefficient(kl, basis.enumerate_multi_indices(5, 2))
    assert np.allclose(np.stack([f.values for f in logn.coeff_fields]), g["logn_fields"], rtol=1e-8, atol=1e-10)


def test_kl_separable_equals_dense():
    # separable 1-D Nystrom product == dense Nystrom (non-degenerate ell1 != ell2)
    spec = random_field.CovarianceSpec(sigma_k=0.3, ell1=0.6, ell2=1.1)
    grid = fem.build_grid(8, 0.0, 1.0)
    d = random_field.kl_expand(spec, grid, 6, method="dense")
    s = random_field.kl_expand(spec, grid, 6, method="separable")
    assert np.allclose(d.eigenvalues, s.eigenvalues, rtol=1e-10)
    for a, b in zip(d.mode_fields, s.mode_fields):
        assert np.allclose(a.values, b.values, rtol=1e-7, atol=1e-9)


def test_baseline_config_shapes():
    # SURVEY §8 shared-size table
    expect = {1: (961, 35, 5, 155, (1, 5, 15, 35)), 2: (3969, 84, 7, 420, (1, 7, 28, 84)),
              5: (16129, 495, 9, 3135, (1, 9, 45, 165, 495))}
    for cfg, (n_h, n_xi, n_t, nnz_h, bounds) in expect.items():
        b = build_problem(cfg)
        assert (b.n_h, b.n_xi, b.n_terms) == (n_h, n_xi, n_t)
        assert sum(h.nnz for h in b.triple.matrices) == nnz_h
        assert b.partition.boundaries == bounds
    assert BASELINE_CONFIGS[4].n == 256 and BASELINE_CONFIGS[3].coefficient_degree == 6
