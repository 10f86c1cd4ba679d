"""Full-size solve fixtures for the headline configurations, produced by the
REFERENCE implementation (`sgkkt`, /root/reference/pkg/src) on this repo's
BASELINE-config inputs (host producers pinned in tests/test_host_producers.py
and tests/test_oracle_golden.py).

    python tests/golden/make_solves.py cfg5 1e-2      # one job per process
    python tests/golden/make_solves.py cfg3 924
    python tests/golden/make_solves.py all            # everything, sequential

Jobs (VERDICT r01 "Next round" item 1):

* cfg5 (128^2 grid, n_xi = 495, n_t = 9), beta in {1e-2, 1e-4, 1e-6}:
  - hGSoc-FGMRES: the reference's own `krylov.fgmres` with its
    `CoupledSweepPreconditioner` (build_coupled_preconditioner) through the
    reference bench seam `bench._steady_callables` (src/bench.py:270-290,
    src/krylov.py:45-137, src/preconditioners.py:411-462);
  - block-diagonal MINRES: the reference's `steady_kkt_apply` and
    `SteadyKKTPreconditioner` (cheb5 mass solves, hGS-Richardson-1 Schur
    block, src/preconditioners.py:227-275) driven by the oracle's MINRES
    restatement (`oracle.minres`; the reference has no MINRES).
* cfg3 (64^2 grid, lognormal Hermite, n_t = 924) hGS-CG for
  n_tau in {1, 7, 924}: the reference's `_build_sweep` (src/preconditioners.py:211-224)
  and `kron_apply` (src/operators.py:88-96) driven by `oracle.cg`.

A solution is far too large to commit (cfg5: 3 x 16129 x 495 doubles), so
each fixture stores the iteration count, the residual history, the true
relative residual, and fingerprints of every (n_h, n_xi) solution block:
its 2-norm, its inner products with four seeded N(0,1) probe matrices
(`probe(k, shape)` below — the GPU tests regenerate them), and two full row
slabs (rows [0, 4) and [n_h/2, n_h/2 + 4)).  The GPU tests compare their own
solve against these at the north-star tolerances (iterations +-1, solution
1e-8 relative).  FGMRES runs with max_iters=60 (the reference preallocates
max_iters+1 basis vectors: 500 would be 89 GB at cfg5; every solve here
converges in < 15 iterations, so the cap never binds).  Run time on one core: ~10-15 min per cfg5 job.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "solves"
SEED = 20240817
SLAB = 4
sys.path.insert(0, str(ROOT))


def probe(k: int, shape) -> np.ndarray:
    return np.random.default_rng(SEED + 1000 + k).standard_normal(shape)


def fingerprint(prefix: str, block: np.ndarray, out: dict) -> None:
    n_h = block.shape[0]
    out[prefix + "_norm"] = np.array(np.linalg.norm(block))
    out[prefix + "_proj"] = np.array([float(np.sum(block * probe(k, block.shape))) for k in range(4)])
    out[prefix + "_slab0"] = block[:SLAB].copy()
    out[prefix + "_slab1"] = block[n_h // 2:n_h // 2 + SLAB].copy()


def _ref():
    if not REF.exists():
        raise SystemExit("reference tree not found; the fixtures are generated in the build container")
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(ROOT))
    import sgkkt.basis as rb
    import sgkkt.bench as rbench
    import sgkkt.krylov as rk
    import sgkkt.operators as ro
    import sgkkt.preconditioners as rp

    return rb, rbench, rk, ro, rp


def _ref_system(bundle, beta):
    """The reference's SteadyKKT / TripleProductSet / LevelPartition built
    from this repo's BASELINE-config matrices (same CSR objects)."""
    rb, rbench, rk, ro, rp = _ref()
    tr = bundle.triple
    triple = rb.TripleProductSet(matrices=list(tr.matrices), variance_penalty=tr.variance_penalty,
                                 objective_weight=tr.objective_weight, gamma=tr.gamma)
    sys_ = ro.SteadyKKT(mass=bundle.mass, stiffness=list(bundle.stiffness), triple=triple, beta=beta,
                        gamma=bundle.spec.gamma, target=bundle.target())
    part = rb.LevelPartition(boundaries=tuple(bundle.partition.boundaries))
    return sys_, part


def _unpack_f(v, n_h, n_xi):
    """Reference packing (F-order matricize per block) -> three (n_h, n_xi) blocks."""
    size = n_h * n_xi
    return [v[i * size:(i + 1) * size].reshape(n_xi, n_h).T for i in range(3)]


def job_cfg5(beta: float) -> None:
    import oracle
    from paper_2512_23804_b200.problems import build_problem

    rb, rbench, rk, ro, rp = _ref()
    bundle = build_problem(5, beta=beta)
    sys_, part = _ref_system(bundle, beta)
    n_h, n_xi = sys_.n_h, sys_.n_xi
    out = {"beta": np.array(beta), "n_h": np.array(n_h), "n_xi": np.array(n_xi)}

    t0 = time.perf_counter()
    soc = rp.build_coupled_preconditioner(sys_, part)
    apply_op, apply_prec, rhs = rbench._steady_callables(sys_, soc)
    out["soc_setup_s"] = np.array(time.perf_counter() - t0)
    t0 = time.perf_counter()
    x, rep = rk.fgmres(apply_op, apply_prec, rhs, rk.FgmresConfig(tol=1e-8, max_iters=60))
    out["soc_seconds"] = np.array(time.perf_counter() - t0)
    out["soc_iters"] = np.array(rep.iterations)
    out["soc_converged"] = np.array(rep.converged)
    out["soc_hist"] = np.asarray(rep.residual_history)
    out["soc_true_res"] = np.array(np.linalg.norm(rhs - apply_op(x)) / np.linalg.norm(rhs))
    for name, blk in zip("yul", _unpack_f(x, n_h, n_xi)):
        fingerprint(f"soc_{name}", blk, out)
    print(f"cfg5 beta={beta:g} hGSoc-FGMRES: {rep.iterations} its, {out['soc_seconds']:.1f} s", flush=True)

    t0 = time.perf_counter()
    bd = rp.build_steady_preconditioner(sys_, part, mass_solver="cheb5", n_tau=sys_.n_terms)
    apply_op, apply_prec, rhs = rbench._steady_callables(sys_, bd)
    out["bd_setup_s"] = np.array(time.perf_counter() - t0)
    t0 = time.perf_counter()
    x, its, conv, hist = oracle.minres(apply_op, apply_prec, rhs, 1e-8)
    out["bd_seconds"] = np.array(time.perf_counter() - t0)
    out["bd_iters"] = np.array(its)
    out["bd_converged"] = np.array(conv)
    out["bd_hist"] = np.asarray(hist)
    out["bd_true_res"] = np.array(np.linalg.norm(rhs - apply_op(x)) / np.linalg.norm(rhs))
    for name, blk in zip("yul", _unpack_f(x, n_h, n_xi)):
        fingerprint(f"bd_{name}", blk, out)
    print(f"cfg5 beta={beta:g} blockdiag-MINRES: {its} its, {out['bd_seconds']:.1f} s", flush=True)
    OUT.mkdir(exist_ok=True)
    np.savez_compressed(OUT / f"cfg5_beta{beta:g}.npz", **out)


def job_cfg3(n_tau: int) -> None:
    import oracle
    from paper_2512_23804_b200.problems import build_problem

    rb, rbench, rk, ro, rp = _ref()
    bundle = build_problem(3)
    n_h, n_xi = bundle.n_h, bundle.n_xi
    cp = list(bundle.triple.matrices[: bundle.n_terms])
    part = rb.LevelPartition(boundaries=tuple(bundle.partition.boundaries))
    op, sweep = rp._build_sweep(cp, list(bundle.stiffness), part, n_tau)
    rhs = bundle.forward_rhs()
    shape = (n_h, n_xi)
    t0 = time.perf_counter()
    x, its, conv, hist = oracle.cg(lambda v: ro.kron_apply(op, v.reshape(shape)).ravel(),
                                   lambda v: sweep.apply(v.reshape(shape)).ravel(), rhs.ravel(), 1e-8)
    out = {"n_tau": np.array(n_tau), "n_h": np.array(n_h), "n_xi": np.array(n_xi)}
    out["seconds"] = np.array(time.perf_counter() - t0)
    out["iters"] = np.array(its)
    out["converged"] = np.array(conv)
    out["hist"] = np.asarray(hist)
    out["true_res"] = np.array(np.linalg.norm(rhs.ravel() - ro.kron_apply(op, x.reshape(shape)).ravel())
                               / np.linalg.norm(rhs))
    fingerprint("x", x.reshape(shape), out)
    print(f"cfg3 n_tau={n_tau} hGS-CG: {its} its, {out['seconds']:.1f} s", flush=True)
    OUT.mkdir(exist_ok=True)
    np.savez_compressed(OUT / f"cfg3_tau{n_tau}.npz", **out)


if __name__ == "__main__":
    args = sys.argv[1:] or ["all"]
    if args[0] == "cfg5":
        job_cfg5(float(args[1]))
    elif args[0] == "cfg3":
        job_cfg3(int(args[1]))
    else:
        for b in (1e-2, 1e-4, 1e-6):
            job_cfg5(b)
        for t in (1, 7, 924):
            job_cfg3(t)
