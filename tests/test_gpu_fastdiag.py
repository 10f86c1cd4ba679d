"""Fast-diagonalisation lead solves on the B200 against
the reference's own algorithm (SuperLU lead solves inside the oracle's hGS /
hGSoc sweeps and Krylov drivers).

The modal solve is a different backward-stable algorithm than the LU, so
the per-solve tolerance is stated against the LU result: 1e-11 relative
(2-norm) for the leads and for P~ at beta >= 1e-4, 1e-9 at beta = 1e-6
where P~ itself is ill-conditioned (the LU's own residual there is ~5e-10).
Krylov bar as for every solver here: iteration counts +-1, solutions 1e-8."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import oracle

pytestmark = pytest.mark.gpu

SEED = 20240817


def _rel2(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _segs(rhs, n_seg, width, col0, ld):
    """Row segments as strided views (col0 offset, ld > width) like the
    sweeps pass them."""
    import torch

    rows = rhs.shape[0] // n_seg
    out = []
    for i in range(n_seg):
        buf = torch.zeros((rows, ld), dtype=torch.float64, device="cuda")
        buf[:, col0:col0 + width] = torch.as_tensor(rhs[i * rows:(i + 1) * rows])
        out.append(buf)
    return out


@pytest.mark.parametrize("cfg,n,shifted", [(1, None, False), (5, None, True)])
def test_lead_solve_vs_superlu(cfg, n, shifted):
    import torch

    from paper_2512_23804_b200.fastdiag import fastdiag_factor
    from paper_2512_23804_b200.preconditioners import shifted_lead_terms
    from paper_2512_23804_b200.problems import build_problem, steady_system

    b = build_problem(cfg, n=n)
    a = shifted_lead_terms(steady_system(b))[0] if shifted else b.stiffness[0]
    f = fastdiag_factor(a, b.mass)
    lu = oracle.splu_ref(a)
    rng = np.random.default_rng(SEED)
    for width, col0, ld in ((1, 0, 1), (7, 3, 16), (120, 5, 130)):
        rhs = rng.standard_normal((a.shape[0], width))
        want = lu.solve(rhs)
        (bt,) = _segs(rhs, 1, width, col0, ld)
        xt = torch.full_like(bt, 7.0)
        f.solve_segments([(bt, col0)], [(xt, col0)], width)
        assert _rel2(xt[:, col0:col0 + width], want) <= 1e-11, width
        # columns outside the view untouched
        assert float(xt[:, :col0].sub(7.0).abs().max() if col0 else 0.0) == 0.0
    # host API (LUFactors.solve contract): vector and matrix right-hand sides
    v = rng.standard_normal(a.shape[0])
    assert _rel2(f.solve(v), lu.solve(v)) <= 1e-11


@pytest.mark.parametrize("cfg,n,beta,tol", [(2, None, 1e-2, 1e-11), (5, None, 1e-2, 1e-11),
                                            (5, None, 1e-4, 1e-11), (5, None, 1e-6, 1e-9)])
def test_ptilde_solve_vs_superlu(cfg, n, beta, tol):
    import torch

    from paper_2512_23804_b200.fastdiag import fastdiag_kkt_factor
    from paper_2512_23804_b200.preconditioners import deterministic_kkt_matrix
    from paper_2512_23804_b200.problems import build_problem, steady_system

    b = build_problem(cfg, n=n, beta=beta)
    sys_ = steady_system(b)
    kkt = deterministic_kkt_matrix(sys_)
    lu = spla.splu(kkt.tocsc(), diag_pivot_thresh=1.0)
    f = fastdiag_kkt_factor(sys_.stiffness[0], sys_.mass, sys_.beta)
    rng = np.random.default_rng(SEED)
    for width, col0, ld in ((1, 0, 1), (36, 8, 84), (330, 165, 495)):
        if cfg == 2 and width > 84:
            continue
        rhs = rng.standard_normal((kkt.shape[0], width))
        want = lu.solve(rhs)
        segs = _segs(rhs, 3, width, col0, ld)
        f.solve_segments([(s, col0) for s in segs], [(s, col0) for s in segs], width)  # in place
        got = np.concatenate([s[:, col0:col0 + width].cpu().numpy() for s in segs])
        assert _rel2(got, want) <= tol, (width, _rel2(got, want))


def test_hgsoc_apply_fastdiag_vs_oracle_cfg2():
    from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, deterministic_kkt_matrix
    from paper_2512_23804_b200.problems import build_problem, steady_system

    b = build_problem(2)
    sys_ = steady_system(b)
    soc = build_coupled_preconditioner(sys_, b.partition, lead_solver="fastdiag")
    rng = np.random.default_rng(SEED)
    r = [rng.standard_normal((sys_.n_h, sys_.n_xi)) for _ in range(3)]
    got = soc.apply(*r)
    want = oracle.coupled_sweep_apply(sys_.mass, sys_.stiffness, sys_.triple.matrices, sys_.triple.objective_weight,
                                      sys_.beta, b.partition.boundaries, sys_.n_terms,
                                      oracle.splu_ref(deterministic_kkt_matrix(sys_)), *r)
    g = np.concatenate([x.ravel() for x in got])
    w = np.concatenate([x.ravel() for x in want])
    assert _rel2(g, w) <= 1e-11


def test_forward_hgs_cg_fastdiag_cfg1():
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, cg
    from paper_2512_23804_b200.operators import kron_apply
    from paper_2512_23804_b200.preconditioners import build_sweep
    from paper_2512_23804_b200.problems import build_problem

    b = build_problem(1)
    cp = b.triple.matrices[: b.n_terms]
    op, sweep = build_sweep(cp, b.stiffness, b.partition, b.n_terms, lead_solver="fastdiag", mass=b.mass)
    shape = (b.n_h, b.n_xi)
    rhs = b.forward_rhs()
    x, rep = cg(lambda v: kron_apply(op, v.view(shape)).reshape(-1),
                lambda v: sweep.apply_device(v.view(shape)).reshape(-1),
                torch.as_tensor(rhs.ravel()).cuda(), FgmresConfig(tol=1e-8))
    lu = oracle.splu_ref(b.stiffness[0])
    xo, its, conv, _ = oracle.cg(lambda v: oracle.kron_apply(cp, b.stiffness, v.reshape(shape)).ravel(),
                                 lambda v: oracle.hgs_apply(cp, b.stiffness, b.partition.boundaries, b.n_terms, lu,
                                                            v.reshape(shape)).ravel(),
                                 rhs.ravel(), 1e-8)
    assert rep.converged and conv and abs(rep.iterations - its) <= 1
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-8 * np.linalg.norm(xo)


@pytest.mark.parametrize("cfg,n,beta", [(2, None, 1e-2), (5, 32, 1e-2), (5, 32, 1e-6)])
def test_control_solves_fastdiag_vs_oracle(cfg, n, beta):
    """hGSoc-FGMRES and block-diagonal-hGS MINRES with fast-diagonalisation
    leads against the oracle's SuperLU-based solves."""
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, fgmres, minres
    from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, build_steady_preconditioner

    from test_gpu_configs import _control, _kkt_callables, _oracle_kkt

    b, sys_ = _control(cfg, n=n, beta=beta)
    o_op, o_soc, o_bd, rhs = _oracle_kkt(sys_, b)
    bt = torch.as_tensor(rhs).cuda()
    soc = build_coupled_preconditioner(sys_, b.partition, lead_solver="fastdiag")
    op, pr = _kkt_callables(sys_, soc)
    x, rep = fgmres(op, pr, bt, FgmresConfig(tol=1e-8))
    xo, its, conv, _ = oracle.fgmres(o_op, o_soc, rhs, 1e-8)
    assert rep.converged and conv and abs(rep.iterations - its) <= 1, (rep.iterations, its)
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-8 * np.linalg.norm(xo)
    bd = build_steady_preconditioner(sys_, b.partition, "cheb5", lead_solver="fastdiag")
    op, pr = _kkt_callables(sys_, bd)
    x2, rep2 = minres(op, pr, bt, FgmresConfig(tol=1e-8))
    xo2, its2, conv2, _ = oracle.minres(o_op, o_bd, rhs, 1e-8)
    assert rep2.converged and conv2 and abs(rep2.iterations - its2) <= 1, (rep2.iterations, its2)
    assert np.linalg.norm(x2.cpu().numpy() - xo2) <= 1e-8 * np.linalg.norm(xo2)


def test_stacked_segments_match_separate_segments():
    """P~ solves on the y/u/lambda blocks of one stacked buffer (passes 1 and 4
    batched over all three segments) equal the per-segment path."""
    import torch

    from paper_2512_23804_b200.fastdiag import fastdiag_kkt_factor
    from paper_2512_23804_b200.problems import build_problem, steady_system

    b = build_problem(2)
    sys_ = steady_system(b)
    f = fastdiag_kkt_factor(sys_.stiffness[0], sys_.mass, sys_.beta)
    rng = np.random.default_rng(21)
    stack = torch.as_tensor(rng.standard_normal((3, sys_.n_h, sys_.n_xi))).cuda()
    sep = [stack[i].clone() for i in range(3)]
    for lo, hi in b.partition.ranges():
        f.solve_segments([(stack[i], lo) for i in range(3)], [(stack[i], lo) for i in range(3)], hi - lo)
        f.solve_segments([(t, lo) for t in sep], [(t, lo) for t in sep], hi - lo)
    got = stack.cpu().numpy()
    want = np.stack([t.cpu().numpy() for t in sep])
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
