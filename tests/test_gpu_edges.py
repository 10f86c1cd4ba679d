"""Edge cases on the B200 through the drop-in API, against the oracle:
smallest meshes (one interior node), a single chaos mode, empty and
coupling-free column slices (reference operators.py:119-126 returns zeros),
the widest column count one CTA can hold (the fast path's limit) and beyond
it, truncation n_tau = 1 (identity only: the sweep is a block-Jacobi solve),
Krylov argument errors, max_iters caps and zero right-hand sides
(krylov.py:55-61)."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _rel(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    scale = float(np.abs(b).max())
    return float(np.abs(a - b).max()) / scale if scale > 0 else float(np.abs(a).max())


def _bundle(n, m, p, family="legendre"):
    from paper_2512_23804_b200.problems import ConfigSpec, build_problem

    return build_problem(ConfigSpec("edge", "forward", n, m, p, family, "affine", 0.2, 1.0))


@pytest.mark.parametrize("n,m,p", [(2, 1, 1), (3, 1, 0), (4, 2, 2)])
def test_tiny_meshes_and_single_mode(n, m, p):
    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply, kron_apply_sliced
    from paper_2512_23804_b200.preconditioners import build_sweep

    b = _bundle(n, m, p)
    cp = b.triple.matrices[: b.n_terms]
    op = KroneckerSumOperator(couplings=cp, operators=b.stiffness)
    x = np.random.default_rng(1).standard_normal((b.n_h, b.n_xi))
    assert _rel(kron_apply(op, x), oracle.kron_apply(cp, b.stiffness, x)) <= TOL
    if b.n_xi > 1:
        got = kron_apply_sliced(op, x, (0, 1), (1, b.n_xi), b.n_terms)
        assert _rel(got, oracle.kron_apply_sliced(cp, b.stiffness, x, (0, 1), (1, b.n_xi), b.n_terms)) <= TOL
    _, sweep = build_sweep(cp, b.stiffness, b.partition, b.n_terms)
    lu = oracle.splu_ref(b.stiffness[0])
    assert _rel(sweep.apply(x), oracle.hgs_apply(cp, b.stiffness, b.partition.boundaries, b.n_terms, lu, x)) <= TOL


def test_empty_and_coupling_free_slices_are_zero():
    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply_sliced

    b = _bundle(6, 3, 2)
    cp = b.triple.matrices[: b.n_terms]
    op = KroneckerSumOperator(couplings=cp, operators=b.stiffness)
    x = np.random.default_rng(2).standard_normal((b.n_h, b.n_xi))
    out = kron_apply_sliced(op, x, (2, 2), (0, b.n_xi), b.n_terms)  # empty source
    assert out.shape == (b.n_h, b.n_xi) and not np.any(out)
    out = kron_apply_sliced(op, x, (0, b.n_xi), (3, 3), b.n_terms)  # empty destination
    assert out.shape == (b.n_h, 0)
    # degree-0 input against the top degree level: no H_t entry (degree gap 2)
    lo, hi = b.partition.ranges()[-1]
    out = kron_apply_sliced(op, x, (0, 1), (lo, hi), b.n_terms)
    assert out.shape == (b.n_h, hi - lo) and not np.any(out)
    assert not np.any(oracle.kron_apply_sliced(cp, b.stiffness, x, (0, 1), (lo, hi), b.n_terms))


@pytest.mark.parametrize("n_xi_cols", [4096, 4500])
def test_widest_column_counts(n_xi_cols):
    """The 9-point fast path holds <= 16 gather chunks per warp (4096 output
    columns per CTA); wider programs take the general program kernel.  Random
    sparse symmetric couplings on a 5x5 mesh, both sides of the limit."""
    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply

    b = _bundle(6, 2, 1)  # 25 interior nodes, 3 terms
    rng = np.random.default_rng(3)
    cps = [sp.identity(n_xi_cols, format="csr")]
    for _ in range(b.n_terms - 1):
        h = sp.random(n_xi_cols, n_xi_cols, density=1.0 / n_xi_cols, random_state=rng, format="csr")
        cps.append(((h + h.T) * 0.5).tocsr())
    op = KroneckerSumOperator(couplings=cps, operators=b.stiffness)
    x = rng.standard_normal((b.n_h, n_xi_cols))
    assert _rel(kron_apply(op, x), oracle.kron_apply(cps, b.stiffness, x)) <= TOL


def test_n_tau_one_is_block_jacobi_with_the_lead():
    from paper_2512_23804_b200.preconditioners import build_sweep

    b = _bundle(8, 3, 2)
    cp = b.triple.matrices[: b.n_terms]
    _, sweep = build_sweep(cp, b.stiffness, b.partition, 1)
    x = np.random.default_rng(4).standard_normal((b.n_h, b.n_xi))
    lu = oracle.splu_ref(b.stiffness[0])
    got = sweep.apply(x)
    assert _rel(got, oracle.hgs_apply(cp, b.stiffness, b.partition.boundaries, 1, lu, x)) <= TOL
    assert _rel(got, lu.solve(x)) <= TOL  # no coupling term survives n_tau = 1


def test_krylov_argument_errors_and_caps():
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, cg, fgmres, minres

    with pytest.raises(ValueError):
        FgmresConfig(tol=0.0)
    with pytest.raises(ValueError):
        FgmresConfig(tol=1e-8, max_iters=0)
    n = 50
    rng = np.random.default_rng(5)
    a = rng.standard_normal((n, n))
    spd = torch.as_tensor(a @ a.T + n * np.eye(n)).cuda()
    op = lambda v: spd @ v
    for solver in (fgmres, cg, minres):
        with pytest.raises(ValueError):
            solver(op, None, torch.zeros(n, dtype=torch.float64, device="cuda"), FgmresConfig(tol=1e-8))
        b = torch.as_tensor(rng.standard_normal(n)).cuda()
        x, rep = solver(op, None, b, FgmresConfig(tol=1e-14, max_iters=2))
        assert rep.iterations == 2 and not rep.converged
        x, rep = solver(op, None, b, FgmresConfig(tol=1e-10))
        assert rep.converged
        assert float(torch.linalg.vector_norm(b - op(x)) / torch.linalg.vector_norm(b)) <= 1e-9
    # max_iters is capped by the problem size (krylov.py:61)
    x, rep = fgmres(op, None, b, FgmresConfig(tol=1e-15, max_iters=500))
    assert rep.iterations <= n


@pytest.mark.parametrize("c1,c2,s", [(-0.37, 1.25, 1.0 / 3.0), (0.0, -2.0, 1.0), (-0.0, 0.0, 0.5), (1.5, 0.0, 1.0)])
def test_lincomb3_matches_the_axpby_chain_bitwise(c1, c2, s):
    """The fused MINRES recurrence pass rounds exactly like the axpby chain it
    replaced (zero coefficients skipped the same way; out aliasing x0)."""
    import torch

    from paper_2512_23804_b200.vec import axpby, lincomb3

    g = torch.Generator().manual_seed(5)
    x0, x1, x2 = (torch.randn(100_003, generator=g, dtype=torch.float64).cuda() for _ in range(3))
    want = x0.clone()
    axpby(want, x1, c1, 1.0)
    axpby(want, x2, c2, 1.0)
    axpby(want, None, 0.0, s)
    got = lincomb3(torch.empty_like(x0), x0, c1, x1, c2, x2, s)
    assert torch.equal(got, want)
    inplace = x0.clone()
    lincomb3(inplace, inplace, c1, x1, c2, x2, s)
    assert torch.equal(inplace, want)
    with pytest.raises(Exception):
        lincomb3(x1, x0, c1, x1, c2, x2, s)


def test_launches_follow_torchs_current_stream():
    """The raw current-stream query used on every launch returns the stream a
    `torch.cuda.stream(...)` context selected (launches are stream-ordered
    with the caller's torch work)."""
    import torch

    from paper_2512_23804_b200 import _lib
    from paper_2512_23804_b200.vec import lincomb3

    side = torch.cuda.Stream()
    assert _lib.stream_ptr() == torch.cuda.current_stream().cuda_stream
    x = torch.arange(1000, dtype=torch.float64, device="cuda")
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        assert _lib.stream_ptr() == side.cuda_stream
        y = lincomb3(torch.empty_like(x), x, s=2.0)
    side.synchronize()
    assert torch.equal(y, 2.0 * x)
