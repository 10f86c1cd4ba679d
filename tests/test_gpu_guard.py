"""Out-of-bounds-write and race canaries for the hand-written kernels.

compute-sanitizer (memcheck / racecheck / synccheck) is closed on this GPU
pool ("runs under it have left GPUs needing a reset"; profiles/r02_sanitizer.txt
keeps the refusal), so the kernels are checked the way that message asks:
outputs are views into larger buffers whose margins (rows above and below,
columns left and right) hold a NaN sentinel that must survive every launch
bit for bit; inputs carry NaN margins too, so a read outside the declared
region poisons the result and fails the oracle comparison; and the
sync-free kernels (flag polling, tickets, counters) are run repeatedly on
identical inputs and must give bitwise-identical results (a missed
acquire/release or a lost update shows up as run-to-run differences)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 20240817


def _framed(rows, cols, top=3, left=5, right=7, bottom=4, fill=float("nan")):
    import torch

    big = torch.full((rows + top + bottom, cols + left + right), fill, dtype=torch.float64, device="cuda")
    return big, big[top:top + rows, left:left + cols]


def _margins_intact(big, view_rows, view_cols, top=3, left=5):
    import torch

    m = torch.ones_like(big, dtype=torch.bool)
    m[top:top + view_rows, left:left + view_cols] = False
    return bool(torch.isnan(big[m]).all())


@pytest.mark.parametrize("cfg,n", [(4, 8), (2, 12), (3, 6)])
def test_coupling_kernels_write_only_their_view(cfg, n):
    """9-point WS / alternating kernels (cfg4-, cfg2-shaped programs) and the
    general program kernel (cfg3, 924 terms), NaN-framed input and output."""
    import torch

    import oracle
    from paper_2512_23804_b200.device import run_program
    from paper_2512_23804_b200.operators import KroneckerSumOperator
    from paper_2512_23804_b200.problems import build_problem

    b = build_problem(cfg, n=n)
    cp = b.triple.matrices[: b.n_terms]
    op = KroneckerSumOperator(couplings=cp, operators=b.stiffness)
    x = np.random.default_rng(SEED).standard_normal((b.n_h, b.n_xi))
    xbig, xv = _framed(b.n_h, b.n_xi)
    xv.copy_(torch.as_tensor(x))
    wbig, wv = _framed(b.n_h, b.n_xi)
    prog = op.program([(0, b.n_xi)], (0, b.n_xi), 0, op.n_terms)
    run_program(op.pattern, prog, [(xv, 0)], [(wv, 0)], alpha=[1.0], beta=[0.0])
    torch.cuda.synchronize()
    assert _margins_intact(wbig, b.n_h, b.n_xi)
    ref = oracle.kron_apply(cp, b.stiffness, x)
    got = wv.cpu().numpy()
    assert np.isfinite(got).all()
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("width", [1, 8, 36, 64, 130])
def test_triangular_solves_write_only_their_columns_and_are_deterministic(width):
    """Grouped (narrow) and wide-tiled triangular solves on the config-5-shaped
    P~ (32^2 grid): NaN-framed segments, columns offset inside the view; five
    runs bitwise identical."""
    import torch

    from paper_2512_23804_b200.preconditioners import deterministic_kkt_matrix
    from paper_2512_23804_b200.problems import build_problem, steady_system
    import scipy.sparse.linalg as spla

    from paper_2512_23804_b200 import linalg

    b = build_problem(5, n=32)
    s = steady_system(b)
    k = deterministic_kkt_matrix(s).tocsc()
    lu = spla.splu(k, diag_pivot_thresh=1.0)
    fac = linalg.TriangularFactors.from_superlu(lu)
    n = s.n_h
    col0 = 3
    cols = width + 2 * col0
    rhs = np.random.default_rng(7).standard_normal((3 * n, width))
    frames_b = [_framed(n, cols) for _ in range(3)]
    for i, (_, v) in enumerate(frames_b):
        v[:, col0:col0 + width] = torch.as_tensor(np.ascontiguousarray(rhs[i * n:(i + 1) * n]))
    outs = []
    for _ in range(5):
        frames_x = [_framed(n, cols) for _ in range(3)]
        fac.solve_segments([(v, col0) for _, v in frames_b], [(v, col0) for _, v in frames_x], width)
        torch.cuda.synchronize()
        for big, v in frames_x:
            # everything outside [col0, col0+width) of the view is untouched
            inner = v[:, col0:col0 + width].clone()
            v[:, col0:col0 + width] = float("nan")
            assert bool(torch.isnan(big).all())
            v[:, col0:col0 + width] = inner
        outs.append(torch.cat([v[:, col0:col0 + width] for _, v in frames_x]).cpu().numpy())
    for big, v in frames_b:  # inputs untouched outside (and inside) their region
        assert _margins_intact(big, n, cols)
    want = lu.solve(rhs)
    assert np.linalg.norm(outs[0] - want) <= 1e-11 * np.linalg.norm(want)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("n_seg", [1, 3])
def test_fastdiag_writes_only_its_columns(n_seg):
    import torch

    from paper_2512_23804_b200.fastdiag import fastdiag_factor, fastdiag_kkt_factor
    from paper_2512_23804_b200.problems import build_problem, steady_system

    b = build_problem(5, n=32)
    s = steady_system(b)
    fac = fastdiag_factor(s.stiffness[0], s.mass) if n_seg == 1 else fastdiag_kkt_factor(s.stiffness[0], s.mass, s.beta)
    n = s.n_h
    width, col0 = 45, 2
    cols = width + 5
    rng = np.random.default_rng(3)
    fb = [_framed(n, cols) for _ in range(n_seg)]
    for _, v in fb:
        v[:, col0:col0 + width] = torch.as_tensor(rng.standard_normal((n, width)))
    fx = [_framed(n, cols) for _ in range(n_seg)]
    fac.solve_segments([(v, col0) for _, v in fb], [(v, col0) for _, v in fx], width)
    torch.cuda.synchronize()
    for big, v in fx:
        inner = v[:, col0:col0 + width].clone()
        assert bool(torch.isfinite(inner).all())
        v[:, col0:col0 + width] = float("nan")
        assert bool(torch.isnan(big).all())
