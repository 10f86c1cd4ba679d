"""§8(f) row 1 on the GPU: all-at-once time-dependent KKT operator and the
parallel-in-time preconditioner against the reference's golden vectors."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

from golden_io import load, steady_case

pytestmark = pytest.mark.gpu


def _system():
    from paper_2512_23804_b200.basis import LevelPartition, TripleProductSet
    from paper_2512_23804_b200.operators import SteadyKKT
    from paper_2512_23804_b200.timedep import TimeKKT, build_time_stencil

    c = steady_case("time_affine_n6")
    n_steps = int(load("time_affine_n6")["n_t"])
    n_xi = c["target"].shape[1]
    triple = TripleProductSet(matrices=c["couplings"], variance_penalty=sp.diags((np.arange(n_xi) > 0) * 1.0),
                              objective_weight=sp.diags(c["weight_diag"], format="csr"), gamma=float(c["gamma"]))
    st = SteadyKKT(mass=c["mass"], stiffness=c["stiffness"], triple=triple, beta=float(c["beta"]),
                   gamma=float(c["gamma"]), target=c["target"])
    return c, TimeKKT(steady=st, stencil=build_time_stencil(n_steps), initial_state=c["y0"]), \
        LevelPartition(boundaries=c["boundaries"])


def _rel(a, b):
    return float(np.abs(np.asarray(a) - b).max() / np.abs(b).max())


def test_time_kkt_apply_and_rhs():
    from paper_2512_23804_b200.timedep import time_kkt_apply, time_rhs

    c, sys_, _ = _system()
    assert _rel(time_kkt_apply(sys_, c["v"]), c["kkt"]) <= 1e-12
    assert _rel(time_rhs(sys_), c["rhs"]) <= 1e-14


@pytest.mark.parametrize("which", ["one", "full"])
def test_pint_preconditioner(which):
    from paper_2512_23804_b200.timedep import build_time_preconditioner

    c, sys_, part = _system()
    n_tau = 1 if which == "one" else int(c["n_terms"])
    prec = build_time_preconditioner(sys_, part, mass_solver="cheb5", n_tau=n_tau)
    got = prec.apply(c["v"])
    assert _rel(got, c[f"pint_tau{n_tau}"]) <= 1e-12
    # block diagonal in time: in the per-step loop the step order is
    # irrelevant, bit for bit; the default all-steps-batched path agrees with
    # it to rounding
    inorder = prec.apply(c["v"], step_order=list(range(sys_.n_t)))
    assert np.array_equal(prec.apply(c["v"], step_order=[2, 0, 3, 1]), inorder)
    assert _rel(inorder, c[f"pint_tau{n_tau}"]) <= 1e-12
    assert _rel(got, inorder) <= 1e-13


def test_pint_fgmres_solve_matches_reference():
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, fgmres
    from paper_2512_23804_b200.timedep import (build_time_preconditioner, from_device_layout, time_kkt_apply,
                                               to_device_layout)

    c, sys_, part = _system()
    prec = build_time_preconditioner(sys_, part, mass_solver="cheb5")
    b = to_device_layout(sys_, c["rhs"])
    x, rep = fgmres(lambda v: time_kkt_apply(sys_, v), lambda v: prec.apply(v), b, FgmresConfig(tol=1e-6))
    assert rep.converged and abs(rep.iterations - int(c["fgmres_iters"])) <= 1
    xf = from_device_layout(sys_, x)
    assert np.linalg.norm(xf - c["fgmres_x"]) <= 1e-8 * np.linalg.norm(c["fgmres_x"])


def test_pint_with_fastdiag_leads_matches_reference():
    """The time-shifted lead (1 + tau sqrt((1+gamma)/beta)) M + tau A_1 is a
    Kronecker sum on the reference's tensor grid: the PINT preconditioner with
    the depth-free lead solves reproduces the
    reference's golden output to the fast diagonalisation's rounding and the
    same FGMRES iteration count."""
    import torch

    from paper_2512_23804_b200.fastdiag import FastDiagFactors
    from paper_2512_23804_b200.krylov import FgmresConfig, fgmres
    from paper_2512_23804_b200.timedep import (build_time_preconditioner, from_device_layout, time_kkt_apply,
                                               to_device_layout)

    c, sys_, part = _system()
    n_tau = int(c["n_terms"])
    prec = build_time_preconditioner(sys_, part, mass_solver="cheb5", n_tau=n_tau, lead_solver="fastdiag")
    assert isinstance(prec.sweep.lead_factor, FastDiagFactors)
    assert _rel(prec.apply(c["v"]), c[f"pint_tau{n_tau}"]) <= 1e-11
    b = to_device_layout(sys_, c["rhs"])
    x, rep = fgmres(lambda v: time_kkt_apply(sys_, v), lambda v: prec.apply(v), b, FgmresConfig(tol=1e-6))
    assert rep.converged and abs(rep.iterations - int(c["fgmres_iters"])) <= 1
    xf = from_device_layout(sys_, x)
    assert np.linalg.norm(xf - c["fgmres_x"]) <= 1e-8 * np.linalg.norm(c["fgmres_x"])


def test_batched_mass_solves_equal_per_block_solves():
    """The PINT preconditioner's batched Chebyshev mass solve (all 2 N_t
    blocks per launch) equals the per-block solve bitwise, including a block
    count above the grid's resident warps and a zero-step solve."""
    import torch

    from paper_2512_23804_b200.preconditioners import make_mass_solver
    from paper_2512_23804_b200.problems import build_problem, steady_system

    b = build_problem(2)
    st = steady_system(b)
    ms = make_mass_solver(st.mass, "cheb5", st.pattern, st.mass_slice)
    dm = ms.device_mass
    g = torch.Generator().manual_seed(3)
    stack = torch.randn((5, st.n_h, st.n_xi), generator=g, dtype=torch.float64).cuda()
    for its in (5, 1, 0):
        got = dm.cheb_batched(stack, its)
        for i in range(stack.shape[0]):
            assert torch.equal(got[i], dm.cheb(stack[i], its)), (its, i)


@pytest.mark.parametrize("lead", ["lu", "fastdiag"])
def test_step_batched_schur_block_matches_per_step_loop(lead):
    """All N_t steps' Z^-1 M_gamma Z^-1 as one sweep over interleaved step
    columns (couplings H_t (x) I_{N_t}) against the reference-shaped per-step
    loop: y and u blocks bitwise, the lambda block to rounding."""
    from paper_2512_23804_b200.timedep import build_time_preconditioner

    c, sys_, part = _system()
    prec = build_time_preconditioner(sys_, part, mass_solver="cheb5", n_tau=int(c["n_terms"]), lead_solver=lead)
    batched = prec.apply(c["v"])
    stepwise = prec.apply(c["v"], step_order=list(range(sys_.n_t)))
    n = len(batched) // 3
    assert np.array_equal(batched[:2 * n], stepwise[:2 * n])
    assert _rel(batched[2 * n:], stepwise[2 * n:]) <= 1e-13


def test_interleaved_kkt_matches_per_step_launches():
    """The all-at-once operator as one program on interleaved step columns
    equals the per-step launches to rounding, and the reference's golden
    output at 1e-12."""
    import torch

    from paper_2512_23804_b200.timedep import (from_device_layout, time_kkt_apply_device,
                                               time_kkt_apply_interleaved, to_device_layout)

    c, sys_, _ = _system()
    v = to_device_layout(sys_, c["v"])
    a = time_kkt_apply_device(sys_, v, torch.empty_like(v))
    b = time_kkt_apply_interleaved(sys_, v, torch.empty_like(v))
    assert float((a - b).abs().max()) <= 1e-13 * float(a.abs().max())
    assert _rel(from_device_layout(sys_, b), c["kkt"]) <= 1e-12
