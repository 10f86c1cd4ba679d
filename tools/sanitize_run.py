"""Small driver for compute-sanitizer (racecheck / synccheck / memcheck):
launches every kernel family of the hot path once or twice on tiny inputs
so the sanitizer's per-access instrumentation finishes in minutes.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Kernels exercised: the warp-specialised 9-point coupling kernel (named
barriers; a config-4-shaped program: 8 column groups of the 1001-column
basis on a 6x6 grid), the alternating 9-point kernel (config-2 level
couplings), the general program kernel (config-3 many-term operator), the
sync-free grouped triangular solves (hGSoc apply with SuperLU factors, both
narrow and wide levels, with and without the dense separator streaming),
the fast-diagonalisation lead solve, the Chebyshev step and the
deterministic reductions of FGMRES / MINRES."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_23804_b200 import _lib, linalg  # noqa: E402
from paper_2512_23804_b200.krylov import FgmresConfig, fgmres, minres  # noqa: E402
from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply, steady_kkt_apply_device  # noqa: E402
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, build_steady_preconditioner  # noqa: E402
from paper_2512_23804_b200.problems import build_problem, steady_system  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(1)
    l0 = _lib.launch_count()
    # warp-specialised 9-point kernel: config-4 basis (1001 columns, 8 groups)
    b4 = build_problem(4, n=6)
    op4 = KroneckerSumOperator(couplings=b4.triple.matrices[: b4.n_terms], operators=b4.stiffness)
    kron_apply(op4, torch.as_tensor(rng.standard_normal((b4.n_h, b4.n_xi))).cuda())
    # general program kernel: config-3 many-term operator
    b3 = build_problem(3, n=5)
    op3 = KroneckerSumOperator(couplings=b3.triple.matrices[: b3.n_terms], operators=b3.stiffness)
    kron_apply(op3, torch.as_tensor(rng.standard_normal((b3.n_h, b3.n_xi))).cuda())
    # control problem: KKT matvec, hGSoc (grouped triangular solves), block-diag MINRES
    b2 = build_problem(2, n=12)
    s2 = steady_system(b2)
    n = s2.block_size()
    shape = (s2.n_h, s2.n_xi)
    rhs = np.zeros(3 * n)
    rhs[:n] = np.asarray(s2.mass @ s2.target).ravel()
    bt = torch.as_tensor(rhs).cuda()

    def split(v):
        return [v[i * n:(i + 1) * n].view(shape) for i in range(3)]

    def op(v):
        o = torch.empty_like(v)
        steady_kkt_apply_device(s2, *split(v), tuple(split(o)))
        return o

    for dense in (True, False):
        linalg.DENSE = dense
        for lead in ("lu", "fastdiag"):
            soc = build_coupled_preconditioner(s2, b2.partition, lead_solver=lead)

            def pr(v, soc=soc):
                o = torch.empty_like(v)
                soc.apply_device(*split(v), outs=tuple(split(o)))
                return o

            x, rep = fgmres(op, pr, bt, FgmresConfig(tol=1e-8, max_iters=3))
            print(f"hGSoc-FGMRES dense={dense} lead={lead}: {rep.iterations} its", flush=True)
    bd = build_steady_preconditioner(s2, b2.partition, "cheb5")

    def pb(v):
        o = torch.empty_like(v)
        bd.apply_device(*split(v), outs=tuple(split(o)))
        return o

    x, rep = minres(op, pb, bt, FgmresConfig(tol=1e-8, max_iters=3))
    print(f"block-diag MINRES: {rep.iterations} its", flush=True)
    torch.cuda.synchronize()
    print(f"sanitize_run ok: {_lib.launch_count() - l0} launches", flush=True)


if __name__ == "__main__":
    main()
