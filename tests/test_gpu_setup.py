"""GPU setup pipeline against the host setup, which is
pinned to the reference (tests/test_host_producers.py): device-assembled
stiffness / mass slices and lognormal coefficient fields agree with the host
assembly to rounding (the element sums are the same, the Gauss-point sum
order inside an element may differ: 1e-14 relative), the operators built on
them reuse the device pattern, and products / solves on them match the
oracle run on the host-assembled matrices."""

from __future__ import annotations

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _maxrel(a, b):
    d = abs(a - b).max()
    return float(d / abs(b).max())


@pytest.mark.parametrize("cfg,n", [(1, None), (2, 24), (3, 16)])
def test_device_assembly_matches_host(cfg, n):
    from paper_2512_23804_b200.gpu_setup import build_problem_device
    from paper_2512_23804_b200.problems import build_problem

    h = build_problem(cfg, n=n)
    d = build_problem_device(cfg, n=n)
    assert d.n_terms == h.n_terms and d.n_h == h.n_h
    for a, b in zip(d.stiffness, h.stiffness):
        assert (a.indptr == b.indptr).all() and (a.indices == b.indices).all()
        assert _maxrel(a, b) <= 1e-14
    assert _maxrel(d.mass, h.mass) <= 1e-15
    for fa, fb in zip(d.coefficient.coeff_fields, h.coefficient.coeff_fields):
        assert np.abs(fa.values - fb.values).max() <= 1e-14 * max(np.abs(fb.values).max(), 1e-300)


def test_device_pattern_reused_and_products_match_oracle():
    from paper_2512_23804_b200.gpu_setup import build_problem_device
    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply, steady_kkt_apply
    from paper_2512_23804_b200.problems import build_problem, steady_system

    d = build_problem_device(3, n=16)
    h = build_problem(3, n=16)
    cp = d.triple.matrices[: d.n_terms]
    op = KroneckerSumOperator(couplings=cp, operators=d.stiffness)
    assert op.pattern is d.extras["device_pattern"]
    x = np.random.default_rng(11).standard_normal((d.n_h, d.n_xi))
    want = oracle.kron_apply(cp, h.stiffness, x)
    assert np.abs(kron_apply(op, x) - want).max() <= 1e-12 * np.abs(want).max()
    d2 = build_problem_device(2, n=24)
    h2 = build_problem(2, n=24)
    sd, sh = steady_system(d2), steady_system(h2)
    assert sd.pattern is d2.extras["device_pattern"]
    rng = np.random.default_rng(12)
    blocks = [rng.standard_normal((sd.n_h, sd.n_xi)) for _ in range(3)]
    got = steady_kkt_apply(sd, *blocks)
    want = oracle.steady_kkt_apply(sh.mass, sh.stiffness, sh.triple.matrices[: sh.n_terms],
                                   sh.triple.weight_diagonal, sh.beta, *blocks)
    for g, w in zip(got, want):
        assert np.abs(g - w).max() <= 1e-12 * np.abs(w).max()


def test_forward_cg_on_device_setup():
    import torch

    from paper_2512_23804_b200.gpu_setup import build_problem_device
    from paper_2512_23804_b200.krylov import FgmresConfig, cg
    from paper_2512_23804_b200.operators import kron_apply
    from paper_2512_23804_b200.preconditioners import build_sweep
    from paper_2512_23804_b200.problems import build_problem

    d = build_problem_device(3, n=16)
    h = build_problem(3, n=16)
    cp = d.triple.matrices[: d.n_terms]
    op, sweep = build_sweep(cp, d.stiffness, d.partition, 7)
    shape = (d.n_h, d.n_xi)
    rhs = h.forward_rhs()
    x, rep = cg(lambda v: kron_apply(op, v.view(shape)).reshape(-1),
                lambda v: sweep.apply_device(v.view(shape)).reshape(-1),
                torch.as_tensor(rhs.ravel()).cuda(), FgmresConfig(tol=1e-8))
    lu = oracle.splu_ref(h.stiffness[0])
    xo, its, conv, _ = oracle.cg(lambda v: oracle.kron_apply(cp, h.stiffness, v.reshape(shape)).ravel(),
                                 lambda v: oracle.hgs_apply(cp, h.stiffness, h.partition.boundaries, 7, lu,
                                                            v.reshape(shape)).ravel(), rhs.ravel(), 1e-8)
    assert rep.converged and conv and abs(rep.iterations - its) <= 1
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-8 * np.linalg.norm(xo)
