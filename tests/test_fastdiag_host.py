"""Fast-diagonalisation lead solves, host side (CPU):
the Kronecker-sum detection on the BASELINE matrices, its refusals, and the
modal algebra the CUDA path implements (a NumPy model of the four passes and
the 3x3 modal solve) against SuperLU — the reference's own lead solve."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
from paper_2512_23804_b200 import fastdiag
from paper_2512_23804_b200.preconditioners import deterministic_kkt_matrix, shifted_lead_terms
from paper_2512_23804_b200.problems import build_problem, steady_system


def _passes(s, lam_fn, segs, n):
    """NumPy model of csrc/fastdiag.cu: T^T on every segment (pass 1 along
    ix, pass 2 along iy), the modal solve, T on the way back."""
    w = segs[0].shape[1]
    fwd = [np.einsum("ia,jb,ijk->abk", s, s, g.reshape(n, n, w)).reshape(n * n, w) for g in segs]
    mod = lam_fn(fwd)
    return [np.einsum("ia,jb,abk->ijk", s, s, g.reshape(n, n, w)).reshape(n * n, w) for g in mod]


@pytest.mark.parametrize("cfg,n", [(1, None), (2, 24)])
def test_split_reconstructs_baseline_leads(cfg, n):
    b = build_problem(cfg, n=n)
    k1, m1 = fastdiag.kron_sum_split(b.stiffness[0], b.mass)
    side = int(round(np.sqrt(b.n_h)))
    assert k1.shape == m1.shape == (side, side)
    # 1-D Q1 on a uniform grid: tridiagonal, symmetric
    assert np.abs(np.triu(m1, 2)).max() == 0.0 and np.abs(np.triu(k1, 2)).max() == 0.0
    rec = sp.kron(sp.csr_matrix(k1), m1) + sp.kron(sp.csr_matrix(m1), k1)
    assert abs(rec - b.stiffness[0]).max() <= 1e-13 * abs(b.stiffness[0]).max()


def test_split_accepts_shifted_lead_and_refuses_variable_coefficients():
    b = build_problem(2, n=16)
    sys_ = steady_system(b)
    lead = shifted_lead_terms(sys_)[0]  # A_1 + sqrt((1+gamma)/beta) M
    assert fastdiag.is_kron_sum(lead, b.mass)
    # a KL mode term has a spatially varying coefficient: never a Kronecker sum
    assert not fastdiag.is_kron_sum(b.stiffness[1], b.mass)
    with pytest.raises(ValueError, match="Kronecker"):
        fastdiag.kron_sum_split(b.stiffness[1], b.mass)
    with pytest.raises(ValueError, match="tensor grid"):
        fastdiag.kron_sum_split(sp.identity(12, format="csr"), sp.identity(12, format="csr"))
    with pytest.raises(ValueError):
        fastdiag.kron_sum_split(b.stiffness[0], b.mass[:-1, :-1])


@pytest.mark.parametrize("shifted", [False, True])
def test_modal_model_matches_superlu_lead(shifted):
    b = build_problem(2, n=20)
    sys_ = steady_system(b)
    a = shifted_lead_terms(sys_)[0] if shifted else b.stiffness[0]
    k1, m1 = fastdiag.kron_sum_split(a, b.mass)
    import scipy.linalg

    mu, s = scipy.linalg.eigh(k1, m1)
    n = len(mu)
    lam = (mu[:, None] + mu[None, :]).reshape(-1, 1)
    rng = np.random.default_rng(3)
    rhs = rng.standard_normal((n * n, 5))
    got = _passes(s, lambda f: [f[0] / lam], [rhs], n)[0]
    want = oracle.splu_ref(a).solve(rhs)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("beta", [1e-2, 1e-6])
def test_modal_model_matches_superlu_ptilde(beta):
    b = build_problem(2, n=20, beta=beta)
    sys_ = steady_system(b)
    k1, m1 = fastdiag.kron_sum_split(b.stiffness[0], b.mass)
    import scipy.linalg

    mu, s = scipy.linalg.eigh(k1, m1)
    n = len(mu)
    lam = (mu[:, None] + mu[None, :]).reshape(-1, 1)

    def modal3(f):
        r1, r2, r3 = f
        d = 1.0 / (1.0 + beta * lam * lam)
        return [d * (r1 + lam * (r2 - beta * r3)), d * (lam * (r1 + lam * r2) + r3), d * (r2 - beta * (lam * r1 + r3))]

    rng = np.random.default_rng(4)
    rows = n * n
    rhs = rng.standard_normal((3 * rows, 4))
    got = np.concatenate(_passes(s, modal3, [rhs[i * rows:(i + 1) * rows] for i in range(3)], n))
    kkt = deterministic_kkt_matrix(sys_)
    want = spla.splu(kkt.tocsc(), diag_pivot_thresh=1.0).solve(rhs)
    assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
    # backward error of the modal solve on the P~ the reference factors
    assert np.linalg.norm(kkt @ got - rhs) <= 1e-9 * np.linalg.norm(rhs)


def test_factor_objects_and_argument_checks():
    b = build_problem(1, n=10)
    f = fastdiag.fastdiag_factor(b.stiffness[0], b.mass)
    assert f.shape == b.stiffness[0].shape and f.n_seg == 1 and f.device_factors is f
    assert np.all(f.lam > 0)
    sys_ = steady_system(build_problem(2, n=10))
    g = fastdiag.fastdiag_kkt_factor(sys_.stiffness[0], sys_.mass, sys_.beta)
    assert g.shape == (3 * sys_.n_h, 3 * sys_.n_h) and g.n_seg == 3
    with pytest.raises(ValueError, match="beta"):
        fastdiag.fastdiag_kkt_factor(sys_.stiffness[0], sys_.mass, 0.0)
    from paper_2512_23804_b200.preconditioners import build_sweep

    with pytest.raises(ValueError, match="mass"):
        build_sweep(b.triple.matrices[: b.n_terms], b.stiffness, b.partition, b.n_terms, lead_solver="fastdiag")
    with pytest.raises(ValueError, match="unknown lead solver"):
        build_sweep(b.triple.matrices[: b.n_terms], b.stiffness, b.partition, b.n_terms, lead_solver="qr")
