"""SuperLU on a nested-dissection grid ordering (lead_solver="lu_nd") on the
B200: the same lead solves as the reference's COLAMD factors up to rounding
(1e-12 relative, max-norm), sweeps against the oracle, Krylov counts +-1."""

from __future__ import annotations

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.parametrize("cfg", [1, 5])
def test_nd_lead_solves_match_colamd(cfg):
    from paper_2512_23804_b200.linalg import sparse_lu
    from paper_2512_23804_b200.preconditioners import shifted_lead_terms
    from paper_2512_23804_b200.problems import build_problem, steady_system

    b = build_problem(cfg)
    a = b.stiffness[0] if cfg == 1 else shifted_lead_terms(steady_system(b))[0]
    f = sparse_lu(a, ordering="nd")
    rng = np.random.default_rng(3)
    for width in (1, 7, 120):
        rhs = rng.standard_normal((a.shape[0], width))
        assert _rel(f.solve(rhs), oracle.splu_ref(a).solve(rhs)) <= 1e-12


def test_nd_hgs_sweep_cfg3_full():
    from paper_2512_23804_b200.preconditioners import build_sweep
    from paper_2512_23804_b200.problems import build_problem

    b = build_problem(3)
    cp = b.triple.matrices[: b.n_terms]
    _, sweep = build_sweep(cp, b.stiffness, b.partition, b.n_terms, lead_solver="lu_nd")
    x = np.random.default_rng(5).standard_normal((b.n_h, b.n_xi))
    lu = oracle.splu_ref(b.stiffness[0])
    assert _rel(sweep.apply(x), oracle.hgs_apply(cp, b.stiffness, b.partition.boundaries, b.n_terms, lu, x)) <= 1e-12


@pytest.mark.parametrize("cfg,n", [(2, None), (5, 32)])
def test_nd_blockdiag_minres(cfg, n):
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, minres
    from paper_2512_23804_b200.preconditioners import build_steady_preconditioner

    from test_gpu_configs import _control, _kkt_callables, _oracle_kkt

    b, sys_ = _control(cfg, n=n)
    o_op, _, o_bd, rhs = _oracle_kkt(sys_, b)
    bd = build_steady_preconditioner(sys_, b.partition, "cheb5", lead_solver="lu_nd")
    op, pr = _kkt_callables(sys_, bd)
    x, rep = minres(op, pr, torch.as_tensor(rhs).cuda(), FgmresConfig(tol=1e-8))
    xo, its, conv, _ = oracle.minres(o_op, o_bd, rhs, 1e-8)
    assert rep.converged and conv and abs(rep.iterations - its) <= 1
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-8 * np.linalg.norm(xo)


@pytest.mark.parametrize("cfg,n", [(2, None), (5, 32)])
def test_threshold_pivoting_hgsoc_fgmres(cfg, n):
    """lead_solver="lu_tp": SuperLU threshold partial pivoting (0.01) for P~ —
    the hGSoc apply agrees with the oracle's partial-pivoting LU to rounding
    (1e-11, 2-norm) and FGMRES needs the same iterations (+-1)."""
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, fgmres
    from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner

    from test_gpu_configs import _control, _kkt_callables, _oracle_kkt

    b, sys_ = _control(cfg, n=n)
    o_op, o_soc, _, rhs = _oracle_kkt(sys_, b)
    soc = build_coupled_preconditioner(sys_, b.partition, lead_solver="lu_tp")
    rng = np.random.default_rng(9)
    r = rng.standard_normal(3 * sys_.block_size())
    size = sys_.block_size()
    blocks = [r[i * size:(i + 1) * size].reshape(sys_.n_h, sys_.n_xi) for i in range(3)]
    got = np.concatenate([g.ravel() for g in soc.apply(*blocks)])
    want = o_soc(r)
    assert np.linalg.norm(got - want) <= 1e-11 * np.linalg.norm(want)
    op, pr = _kkt_callables(sys_, soc)
    x, rep = fgmres(op, pr, torch.as_tensor(rhs).cuda(), FgmresConfig(tol=1e-8))
    xo, its, conv, _ = oracle.fgmres(o_op, o_soc, rhs, 1e-8)
    assert rep.converged and conv and abs(rep.iterations - its) <= 1
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-8 * np.linalg.norm(xo)
