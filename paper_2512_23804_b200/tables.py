"""Result tables in the reference's exact schema, so GPU
and CPU rows are diffable line by line.

Mirrors `sgkkt.bench` (reference pkg/src/sgkkt/bench.py):
* `ResultRow` — the row fields (bench.py:236-251);
* `emit_table` — fixed column order and cell formatting, CSV or markdown,
  ValueError on no rows / unknown format (bench.py:366-419);
* `experiment_rows` — the steady-problem experiment loop of `run_experiment`
  (bench.py:325-363: one row per (mass_solver, n_tau), FGMRES with the
  block-diagonal preconditioner, final_rel_res = last recorded residual),
  run on the GPU path.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

__all__ = ["COLUMNS", "ResultRow", "emit_table", "experiment_rows"]

COLUMNS = ("problem", "n", "N_h", "m_xi", "p", "N_xi", "sigma", "beta", "tol", "mass_solver", "n_tau", "iters",
           "converged", "seconds", "final_rel_res")


@dataclass(frozen=True)
class ResultRow:
    problem: str
    n: int
    n_h: int
    m_xi: int
    p: int
    n_xi: int
    sigma: float
    beta: float
    tol: float
    mass_solver: str
    n_tau: int
    iterations: int
    converged: bool
    seconds: float
    final_rel_res: float

    def cells(self) -> list[str]:
        g12 = lambda v: format(float(v), ".12g")
        return [self.problem, str(self.n), str(self.n_h), str(self.m_xi), str(self.p), str(self.n_xi),
                g12(self.sigma), g12(self.beta), g12(self.tol), self.mass_solver, str(self.n_tau),
                str(self.iterations), "true" if self.converged else "false", f"{self.seconds:.6f}",
                f"{self.final_rel_res:.6e}"]


def emit_table(rows: list[ResultRow], format: str = "csv") -> str:  # noqa: A002 (reference keyword)
    if not rows:
        raise ValueError("no rows to emit")
    body = [r.cells() for r in rows]
    if format == "csv":
        return "\n".join([",".join(COLUMNS)] + [",".join(c) for c in body]) + "\n"
    if format == "markdown":
        head = "| " + " | ".join(COLUMNS) + " |"
        rule = "|" + "|".join(" --- " for _ in COLUMNS) + "|"
        return "\n".join([head, rule] + ["| " + " | ".join(c) + " |" for c in body]) + "\n"
    raise ValueError(f"unknown table format {format!r}")


def experiment_rows(bundle, mass_solvers=("cheb5",), n_taus=None, tol: float = 1e-8, beta: float | None = None,
                    max_iters: int = 500, lead_solver: str = "lu") -> list[ResultRow]:
    """Steady-problem rows of the reference experiment on the GPU path: for
    every (mass_solver, n_tau), FGMRES to `tol` preconditioned by the
    block-diagonal preconditioner (reference bench.py:293-363).  `bundle` is
    a problems.ProblemBundle of a control configuration."""
    import torch

    from .krylov import FgmresConfig, fgmres
    from .operators import steady_kkt_apply_device
    from .preconditioners import build_steady_preconditioner
    from .problems import steady_system

    sys_ = steady_system(bundle, beta=beta)
    n = sys_.block_size()
    shape = (sys_.n_h, sys_.n_xi)
    rhs = np.zeros(3 * n)
    rhs[:n] = np.asarray(sys_.mass @ sys_.target).ravel()
    b = torch.as_tensor(rhs).cuda()

    def split(v):
        return [v[i * n:(i + 1) * n].view(shape) for i in range(3)]

    def op(v):
        o = torch.empty_like(v)
        steady_kkt_apply_device(sys_, *split(v), tuple(split(o)))
        return o

    taus = list(n_taus) if n_taus is not None else [1, sys_.n_terms]
    rows = []
    spec = bundle.spec
    for ms in mass_solvers:
        for n_tau in taus:
            prec = build_steady_preconditioner(sys_, bundle.partition, ms, n_tau=n_tau, lead_solver=lead_solver)

            def pr(v, prec=prec):
                o = torch.empty_like(v)
                prec.apply_device(*split(v), outs=tuple(split(o)))
                return o

            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, rep = fgmres(op, pr, b, FgmresConfig(tol=tol, max_iters=max_iters))
            torch.cuda.synchronize()
            secs = time.perf_counter() - t0
            hist = np.asarray(rep.residual_history)
            rows.append(ResultRow(problem="steady", n=spec.n, n_h=sys_.n_h, m_xi=spec.m_xi, p=spec.p,
                                  n_xi=sys_.n_xi, sigma=spec.sigma, beta=sys_.beta, tol=tol, mass_solver=ms,
                                  n_tau=n_tau, iterations=rep.iterations, converged=bool(rep.converged),
                                  seconds=secs, final_rel_res=float(hist[-1]) if hist.size else math.nan))
    return rows
