"""GPU parity at the BASELINE.json configurations (full sizes where the CPU
oracle finishes in seconds; size-independent properties otherwise).

Tolerances (north_star): operator / preconditioner outputs 1e-12 relative;
Krylov iteration counts +-1; final solutions 1e-8 relative."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

import oracle

pytestmark = pytest.mark.gpu

SEED = 20240817


def _rel(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _rel2(a, b):
    """Norm-wise relative difference ||a-b||_2/||b||_2 (used for outputs that
    pass through the P~ triangular solves, whose own SuperLU rounding at
    48k unknowns is ~1e-12 relative in the max norm)."""
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _forward(cfg, n=None):
    from paper_2512_23804_b200.preconditioners import build_sweep
    from paper_2512_23804_b200.problems import build_problem

    b = build_problem(cfg, n=n)
    cp = b.triple.matrices[: b.n_terms]
    return b, cp


def _cg_pair(b, cp, n_tau, tol=1e-8):
    """GPU hGS-CG (drop-in API) and the oracle hGS-CG on the same inputs."""
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, cg
    from paper_2512_23804_b200.operators import kron_apply
    from paper_2512_23804_b200.preconditioners import build_sweep

    op, sweep = build_sweep(cp, b.stiffness, b.partition, n_tau)
    shape = (b.n_h, b.n_xi)
    rhs = b.forward_rhs()
    x_d, rep = cg(lambda v: kron_apply(op, v.view(shape)).reshape(-1),
                  lambda v: sweep.apply_device(v.view(shape)).reshape(-1),
                  torch.as_tensor(rhs.ravel()).cuda(), FgmresConfig(tol=tol))
    lu = oracle.splu_ref(b.stiffness[0])
    x_o, its, conv, _ = oracle.cg(lambda v: oracle.kron_apply(cp, b.stiffness, v.reshape(shape)).ravel(),
                                  lambda v: oracle.hgs_apply(cp, b.stiffness, b.partition.boundaries, n_tau, lu,
                                                             v.reshape(shape)).ravel(),
                                  rhs.ravel(), tol)
    return x_d.cpu().numpy(), rep, x_o, its, conv


def test_cfg1_matvec_and_hgs_cg():
    b, cp = _forward(1)
    rng = np.random.default_rng(SEED)
    x = rng.standard_normal((b.n_h, b.n_xi))
    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply

    op = KroneckerSumOperator(couplings=cp, operators=b.stiffness)
    assert _rel(kron_apply(op, x), oracle.kron_apply(cp, b.stiffness, x)) <= 1e-12
    xd, rep, xo, its, conv = _cg_pair(b, cp, b.n_terms)
    assert rep.converged and conv
    assert abs(rep.iterations - its) <= 1
    assert np.linalg.norm(xd - xo) <= 1e-8 * np.linalg.norm(xo)


@pytest.mark.parametrize("n_tau", [1, 7, 924])
def test_cfg3_lognormal_cg_small_grid(n_tau):
    # cfg3 operators (Hermite, lognormal, coefficient degree 6, n_t = 924) on a
    # 16x16 grid so the oracle CG finishes in seconds
    b, cp = _forward(3, n=16)
    xd, rep, xo, its, conv = _cg_pair(b, cp, n_tau)
    assert rep.converged and conv
    assert abs(rep.iterations - its) <= 1
    assert np.linalg.norm(xd - xo) <= 1e-8 * np.linalg.norm(xo)


def test_cfg3_full_matvec_and_sweep():
    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply
    from paper_2512_23804_b200.preconditioners import build_sweep

    b, cp = _forward(3)
    rng = np.random.default_rng(SEED)
    x = rng.standard_normal((b.n_h, b.n_xi))
    op, sweep = build_sweep(cp, b.stiffness, b.partition, b.n_terms)
    assert _rel(kron_apply(op, x), oracle.kron_apply(cp, b.stiffness, x)) <= 1e-12
    lu = oracle.splu_ref(b.stiffness[0])
    assert _rel(sweep.apply(x), oracle.hgs_apply(cp, b.stiffness, b.partition.boundaries, b.n_terms, lu, x)) <= 1e-12


def test_cfg4_matvec_rows_and_properties():
    import torch

    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply

    b, cp = _forward(4)
    op = KroneckerSumOperator(couplings=cp, operators=b.stiffness)
    rng = np.random.default_rng(SEED)
    x = rng.standard_normal((b.n_h, b.n_xi))
    y = rng.standard_normal((b.n_h, b.n_xi))
    xd = torch.as_tensor(x).cuda()
    yd = torch.as_tensor(y).cuda()
    w = kron_apply(op, xd)
    # oracle on row slabs: first rows (boundary stencils), a middle slab, last rows
    for r0, r1 in ((0, 300), (b.n_h // 2 - 150, b.n_h // 2 + 150), (b.n_h - 300, b.n_h)):
        ref = oracle.kron_apply_rows(cp, b.stiffness, x, (r0, r1))
        assert _rel(w[r0:r1], ref) <= 1e-12
    # linearity and symmetry (A_t, H_t symmetric) at full size
    wy = kron_apply(op, yd)
    lin = kron_apply(op, 2.0 * xd - 0.5 * yd)
    assert float((lin - (2.0 * w - 0.5 * wy)).abs().max() / lin.abs().max()) <= 1e-13
    s1 = float((w * yd).sum())
    s2 = float((wy * xd).sum())
    assert abs(s1 - s2) <= 1e-11 * abs(s1)


def _control(cfg, n=None, beta=None):
    from paper_2512_23804_b200.problems import build_problem, steady_system

    b = build_problem(cfg, n=n, beta=beta)
    return b, steady_system(b)


def _kkt_callables(sys_, prec):
    import torch

    from paper_2512_23804_b200.operators import steady_kkt_apply_device

    n = sys_.block_size()
    shape = (sys_.n_h, sys_.n_xi)

    def split(v):
        return [v[i * n:(i + 1) * n].view(shape) for i in range(3)]

    def op(v):
        o = torch.empty_like(v)
        steady_kkt_apply_device(sys_, *split(v), tuple(split(o)))
        return o

    def pr(v):
        o = torch.empty_like(v)
        prec.apply_device(*split(v), outs=tuple(split(o)))
        return o

    return op, pr


def _oracle_kkt(sys_, b):
    n_h, n_xi = sys_.n_h, sys_.n_xi
    size = n_h * n_xi
    cp = sys_.triple.matrices[: sys_.n_terms]
    w = sys_.triple.weight_diagonal

    def unpack(v):
        return [v[i * size:(i + 1) * size].reshape(n_h, n_xi) for i in range(3)]

    def pack(blocks):
        return np.concatenate([np.asarray(x).ravel() for x in blocks])

    op = lambda v: pack(oracle.steady_kkt_apply(sys_.mass, sys_.stiffness, cp, w, sys_.beta, *unpack(v)))
    m = sys_.mass
    a0 = sys_.stiffness[0]
    kkt_lu = oracle.splu_ref(sp.bmat([[m, None, -a0], [None, sys_.beta * m, m], [-a0, m, None]], format="csr"))
    soc = lambda v: pack(oracle.coupled_sweep_apply(m, sys_.stiffness, sys_.triple.matrices,
                                                    sys_.triple.objective_weight, sys_.beta,
                                                    b.partition.boundaries, sys_.n_terms, kkt_lu, *unpack(v)))
    lead = oracle.splu_ref(oracle.shifted_lead(m, sys_.stiffness, sys_.beta, sys_.gamma)[0])
    bd = lambda v: pack(oracle.steady_precond_apply(m, sys_.stiffness, cp, w, sys_.beta, sys_.gamma,
                                                    b.partition.boundaries, sys_.n_terms, lead, *unpack(v)))
    rhs = np.zeros(3 * size)
    rhs[:size] = np.asarray(m @ sys_.target).ravel()
    return op, soc, bd, rhs


@pytest.mark.parametrize("cfg,n", [(2, None), (5, 32)])
def test_control_hgsoc_fgmres_and_minres(cfg, n):
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, fgmres, minres
    from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, build_steady_preconditioner

    b, sys_ = _control(cfg, n=n)
    o_op, o_soc, o_bd, rhs = _oracle_kkt(sys_, b)
    bt = torch.as_tensor(rhs).cuda()
    soc = build_coupled_preconditioner(sys_, b.partition)
    op, pr = _kkt_callables(sys_, soc)
    x, rep = fgmres(op, pr, bt, FgmresConfig(tol=1e-8))
    xo, its, conv, _ = oracle.fgmres(o_op, o_soc, rhs, 1e-8)
    assert rep.converged and conv and abs(rep.iterations - its) <= 1
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-8 * np.linalg.norm(xo)
    bd = build_steady_preconditioner(sys_, b.partition, "cheb5")
    op, pr = _kkt_callables(sys_, bd)
    x2, rep2 = minres(op, pr, bt, FgmresConfig(tol=1e-8))
    xo2, its2, conv2, _ = oracle.minres(o_op, o_bd, rhs, 1e-8)
    assert rep2.converged and conv2 and abs(rep2.iterations - its2) <= 1
    assert np.linalg.norm(x2.cpu().numpy() - xo2) <= 1e-8 * np.linalg.norm(xo2)
    # true residual of the GPU solution
    r = bt - op(x2)
    assert float(torch.linalg.vector_norm(r) / torch.linalg.vector_norm(bt)) <= 2e-8


def test_cfg5_full_size_operator_and_hgsoc_apply():
    import torch

    from paper_2512_23804_b200.operators import steady_kkt_apply
    from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner

    b, sys_ = _control(5)
    o_op, o_soc, _, _ = _oracle_kkt(sys_, b)
    rng = np.random.default_rng(SEED)
    size = sys_.block_size()
    v = rng.standard_normal(3 * size)
    blocks = [v[i * size:(i + 1) * size].reshape(sys_.n_h, sys_.n_xi) for i in range(3)]
    got = np.concatenate([g.ravel() for g in steady_kkt_apply(sys_, *blocks)])
    assert _rel(got, o_op(v)) <= 1e-12
    soc = build_coupled_preconditioner(sys_, b.partition)
    got = np.concatenate([g.ravel() for g in soc.apply(*blocks)])
    want = o_soc(v)
    assert _rel2(got, want) <= 1e-12
    assert _rel(got, want) <= 1e-11


@pytest.mark.parametrize("cfg,n,n_slabs", [(2, None, 1), (2, None, 32), (2, 8, 32), (2, 8, 1000), (1, 6, 3)])
def test_pinned_host_pipeline_matches_device_path(cfg, n, n_slabs):
    """The overlapped slab pipeline for pinned host buffers (the e2e path)
    gives bit-identical results to the device-resident launch: one slab,
    the default 32, slabs thinner than the stencil reach (8^2 grid: 49 rows
    in 32 slabs) and more slabs than rows."""
    import torch

    from paper_2512_23804_b200.operators import KroneckerSumOperator, _pipeline_ok, kron_apply

    b, cp = _forward(cfg, n=n)
    op = KroneckerSumOperator(couplings=cp, operators=b.stiffness)
    assert _pipeline_ok(op)
    x = torch.randn((b.n_h, b.n_xi), dtype=torch.float64).pin_memory()
    out = torch.empty_like(x).pin_memory()
    got = kron_apply(op, x, out=out, n_slabs=n_slabs)
    want = kron_apply(op, x.cuda()).cpu()
    assert got is out
    assert torch.equal(got, want)


def test_pinned_host_non_contiguous_out_and_many_terms():
    """Pinned buffers the pipeline cannot take (a non-contiguous `out`; a
    many-term config-3 operator whose program has no 9-point schedule) go
    through the plain device path and still match it bit for bit."""
    import torch

    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply

    b, cp = _forward(2, n=12)
    op = KroneckerSumOperator(couplings=cp, operators=b.stiffness)
    x = torch.randn((b.n_h, b.n_xi), dtype=torch.float64).pin_memory()
    big = torch.zeros((b.n_h, 2 * b.n_xi), dtype=torch.float64).pin_memory()
    out = big[:, ::2]
    got = kron_apply(op, x, out=out)
    assert torch.equal(got, kron_apply(op, x.cuda()).cpu())
    b3, cp3 = _forward(3, n=8)
    op3 = KroneckerSumOperator(couplings=cp3, operators=b3.stiffness)
    x3 = torch.randn((b3.n_h, b3.n_xi), dtype=torch.float64).pin_memory()
    out3 = torch.empty_like(x3).pin_memory()
    got3 = kron_apply(op3, x3, out=out3)
    assert torch.equal(got3, kron_apply(op3, x3.cuda()).cpu())
    ref = oracle.kron_apply(cp3, b3.stiffness, x3.numpy())
    assert _rel(got3, ref) <= 1e-12


@pytest.mark.parametrize("wide_min", [32, 10**9])
@pytest.mark.parametrize("dense", [True, False])
def test_ptilde_solve_all_chunk_paths_vs_superlu(dense, wide_min, monkeypatch):
    """The grouped triangular solve through every chunk width / CTA shape
    (1, 2, 4 columns; 512- and 256-thread CTAs above width 200) and with /
    without the dense-region streaming, against SuperLU on the same P~."""
    import scipy.sparse.linalg as spla
    import torch

    from paper_2512_23804_b200 import linalg
    from paper_2512_23804_b200.preconditioners import deterministic_kkt_matrix

    monkeypatch.setattr(linalg, "DENSE", dense)
    monkeypatch.setattr(linalg, "WIDE_MIN", wide_min)  # 32: widths >= 32 take the wide-tiled solve
    b, sys_ = _control(5, n=32)
    k = deterministic_kkt_matrix(sys_).tocsc()
    lu = spla.splu(k, diag_pivot_thresh=1.0)
    fac = linalg.TriangularFactors.from_superlu(lu)
    if dense:
        assert fac.gl.dense_nb > 0 and fac.gu.dense_nb > 0
    n = k.shape[0] // 3
    rng = np.random.default_rng(7)
    for width in (1, 7, 33, 64, 65, 250):
        rhs = rng.standard_normal((3 * n, width))
        want = lu.solve(rhs)
        segs = [torch.as_tensor(np.ascontiguousarray(rhs[i * n:(i + 1) * n])).cuda() for i in range(3)]
        outs = [torch.empty_like(s) for s in segs]
        fac.solve_segments([(s, 0) for s in segs], [(o, 0) for o in outs], width)
        got = np.concatenate([o.cpu().numpy() for o in outs])
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err <= 1e-11, (width, err)


def test_cfg5_ptilde_maxnorm_error_is_superlu_level():
    """Why the full-size config-5 hGSoc apply is bounded at 1e-11 in the max
    norm (1e-12 in the 2-norm): the 48,387-unknown P~ is ill-conditioned
    enough that SuperLU's OWN solve differs from a once-refined solution by
    ~1e-12 in the max norm.  The GPU triangular solves (same factors, a
    different but fixed summation order) must land at that same level:
    max-norm error vs the refined solution <= 4x SuperLU's own, and <= 1e-11."""
    import scipy.sparse.linalg as spla
    import torch

    from paper_2512_23804_b200 import linalg
    from paper_2512_23804_b200.preconditioners import deterministic_kkt_matrix

    b, sys_ = _control(5)
    k = deterministic_kkt_matrix(sys_).tocsr()
    lu = spla.splu(k.tocsc(), diag_pivot_thresh=1.0)
    fac = linalg.TriangularFactors.from_superlu(lu)
    n = sys_.n_h
    rng = np.random.default_rng(11)
    for width in (1, 36):
        rhs = rng.standard_normal((3 * n, width))
        x_lu = lu.solve(rhs)
        x_ref = x_lu + lu.solve(rhs - k @ x_lu)  # one step of iterative refinement
        segs = [torch.as_tensor(np.ascontiguousarray(rhs[i * n:(i + 1) * n])).cuda() for i in range(3)]
        outs = [torch.empty_like(s) for s in segs]
        fac.solve_segments([(s, 0) for s in segs], [(o, 0) for o in outs], width)
        x_gpu = np.concatenate([o.cpu().numpy() for o in outs])
        scale = np.abs(x_ref).max()
        err_lu = np.abs(x_lu - x_ref).max() / scale
        err_gpu = np.abs(x_gpu - x_ref).max() / scale
        print(f"width {width}: max-norm rel. error vs refined solution: SuperLU {err_lu:.2e}, GPU {err_gpu:.2e}")
        assert err_gpu <= max(4.0 * err_lu, 1e-13), (width, err_gpu, err_lu)
        assert err_gpu <= 1e-11, (width, err_gpu)
