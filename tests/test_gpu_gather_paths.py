"""The 9-point kernels read the gather's H-coefficients from the kernel
parameter bank when a program has <= 8 distinct coefficients and from shared
memory otherwise (csrc/stencil9.cu: stencil9_grid_kernel, stencil9_kernel).
Both paths against a SciPy evaluation of W = sum_t A_t V H_t
(reference operators.py:88-96), on a config-4-shaped program (grid kernel, 8
column groups) and a config-2-shaped one (alternating kernel)."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n", [(4, 8), (2, 12)])
@pytest.mark.parametrize("distinct", ["few", "many"])
def test_gather_coefficient_paths_match_scipy(cfg, n, distinct):
    import torch

    from paper_2512_23804_b200.device import run_program
    from paper_2512_23804_b200.operators import KroneckerSumOperator
    from paper_2512_23804_b200.problems import build_problem

    b = build_problem(cfg, n=n)
    cps = [sp.csr_matrix(m, copy=True) for m in b.triple.matrices[: b.n_terms]]
    if distinct == "many":  # 13 scale factors per term: far more than 8 distinct coefficients
        for t, m in enumerate(cps):
            m.data = m.data * (1.0 + 0.01 * ((np.arange(m.nnz) + t) % 13))
    op = KroneckerSumOperator(couplings=cps, operators=b.stiffness)
    prog = op.program([(0, b.n_xi)], (0, b.n_xi), 0, op.n_terms)
    f9 = prog.fast9(op.pattern.n_slices)
    assert f9 is not None
    assert (f9.host.n_coef <= 8) == (distinct == "few")
    x = np.random.default_rng(11).standard_normal((b.n_h, b.n_xi))
    xd = torch.as_tensor(x).cuda()
    wd = torch.full_like(xd, float("nan"))
    run_program(op.pattern, prog, [(xd, 0)], [(wd, 0)], alpha=[1.0], beta=[0.0])
    want = sum(sp.csr_matrix(a) @ x @ h for a, h in zip(b.stiffness[: b.n_terms], cps))
    got = wd.cpu().numpy()
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
