"""Generate the golden vectors under tests/golden/ by running the REFERENCE
implementation (`sgkkt`, /root/reference/pkg/src) on small seeded inputs.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

The resulting .npz files are committed; the tests (CPU and GPU) only read
them, so nothing at test time needs the reference tree.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import scipy.sparse as sp

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
SEED = 20240817  # the reference test seed (tests/conftest.py:18-20)


def _ref():
    if not REF.exists():
        raise SystemExit("reference tree not found; golden vectors are generated in the build container")
    sys.path.insert(0, str(REF))
    import sgkkt.basis as basis
    import sgkkt.bench as bench
    import sgkkt.fem as fem
    import sgkkt.krylov as krylov
    import sgkkt.operators as ops
    import sgkkt.preconditioners as pre
    import sgkkt.problems as problems
    import sgkkt.random_field as rf

    return basis, bench, fem, krylov, ops, pre, problems, rf


def csr_parts(prefix, m, out):
    m = sp.csr_matrix(m)
    out[prefix + "_indptr"] = m.indptr.astype(np.int64)
    out[prefix + "_indices"] = m.indices.astype(np.int64)
    out[prefix + "_data"] = m.data
    out[prefix + "_shape"] = np.array(m.shape, dtype=np.int64)


def gen_kron_random():
    basis, bench, fem, krylov, ops, pre, problems, rf = _ref()
    rng = np.random.default_rng(SEED)
    n_h, n_xi, terms = 7, 5, 4
    out = {}
    hs, as_ = [], []
    for t in range(terms):
        h = rng.standard_normal((n_xi, n_xi))
        h = sp.csr_matrix((h + h.T) / 2)
        a = sp.csr_matrix(rng.standard_normal((n_h, n_h)))
        hs.append(h)
        as_.append(a)
        csr_parts(f"H{t}", h, out)
        csr_parts(f"A{t}", a, out)
    x = rng.standard_normal((n_h, n_xi))
    op = ops.KroneckerSumOperator(couplings=hs, operators=as_)
    out["terms"] = np.array(terms)
    out["x"] = x
    out["W"] = ops.kron_apply(op, x)
    out["W_sliced_1_4__2_5_t3"] = ops.kron_apply_sliced(op, x, (1, 4), (2, 5), 3)
    np.savez_compressed(OUT / "kron_random.npz", **out)


def gen_steady(name, n, m_xi, p, coefficient, degree, sigma, beta):
    basis, bench, fem, krylov, ops, pre, problems, rf = _ref()
    rng = np.random.default_rng(SEED + n)
    bundle = problems.build_steady_problem(n=n, m_xi=m_xi, p=p, sigma_k=sigma, beta=beta,
                                           coefficient=coefficient, coefficient_degree=degree)
    sys_ = bundle.system
    out = {"n": np.array(n), "beta": np.array(beta), "gamma": np.array(sys_.gamma),
           "boundaries": np.array(bundle.partition.boundaries, dtype=np.int64)}
    csr_parts("M", sys_.mass, out)
    out["n_terms"] = np.array(sys_.n_terms)
    for t, a in enumerate(sys_.stiffness):
        csr_parts(f"A{t}", a, out)
    for t, h in enumerate(sys_.triple.matrices):
        csr_parts(f"H{t}", h, out)
    out["weight_diag"] = sys_.triple.weight_diagonal
    out["target"] = sys_.target
    shape = (sys_.n_h, sys_.n_xi)
    x = rng.standard_normal(shape)
    r = [rng.standard_normal(shape) for _ in range(3)]
    out["x"] = x
    out["r_y"], out["r_u"], out["r_lam"] = r
    a_op = sys_.stiffness_operator()
    out["W"] = ops.kron_apply(a_op, x)
    for lvl, (lo, hi) in enumerate(bundle.partition.ranges()):
        out[f"before_{lvl}"] = ops.kron_apply_sliced(a_op, x, (0, lo), (lo, hi), a_op.n_terms)
        out[f"after_{lvl}"] = ops.kron_apply_sliced(a_op, x, (hi, shape[1]), (lo, hi), a_op.n_terms)
    out["kkt_y"], out["kkt_u"], out["kkt_lam"] = ops.steady_kkt_apply(sys_, *r)
    out["rhs_y"] = ops.steady_rhs(sys_)[0]
    out["cheb5"] = pre.chebyshev_mass_solve(sys_.mass, r[0], 5)
    for n_tau in sorted({1, 2, sys_.n_terms}):
        prec = pre.build_steady_preconditioner(sys_, bundle.partition, mass_solver="cheb5", n_tau=n_tau)
        out[f"hgs_tau{n_tau}"] = prec.sweep.apply(r[2])
        out[f"rich2_tau{n_tau}"] = pre.richardson_hgs(prec.z_operator, prec.sweep, r[2], 2)
        py, pu, pl = prec.apply(*r)
        out[f"bd_y_tau{n_tau}"], out[f"bd_u_tau{n_tau}"], out[f"bd_lam_tau{n_tau}"] = py, pu, pl
        cp = pre.build_coupled_preconditioner(sys_, bundle.partition, n_tau=n_tau)
        cy, cu, cl = cp.apply(*r)
        out[f"soc_y_tau{n_tau}"], out[f"soc_u_tau{n_tau}"], out[f"soc_lam_tau{n_tau}"] = cy, cu, cl
    # forward-problem sweep with the unshifted lead (configs 1/3 path)
    fop, fsweep = pre._build_sweep(sys_.triple.matrices[: sys_.n_terms], list(sys_.stiffness),
                                   bundle.partition, sys_.n_terms)
    out["fwd_hgs"] = fsweep.apply(x)
    # end-to-end FGMRES solves through the reference bench seam (bench.py:293-324)
    xs, rep = bench.solve_bundle(bundle, "cheb5", sys_.n_terms, 1e-8)
    out["fgmres_bd_x"] = xs
    out["fgmres_bd_iters"] = np.array(rep.iterations)
    out["fgmres_bd_hist"] = rep.residual_history
    cprec = pre.build_coupled_preconditioner(sys_, bundle.partition)
    apply_op, _, rhs = bench._steady_callables(sys_, cprec)
    size = sys_.block_size()

    def apply_prec(v):
        blocks = (ops.matricize(v[:size], *shape), ops.matricize(v[size:2 * size], *shape),
                  ops.matricize(v[2 * size:], *shape))
        return np.concatenate([ops.vectorize(b) for b in cprec.apply(*blocks)])

    xs2, rep2 = krylov.fgmres(apply_op, apply_prec, rhs, krylov.FgmresConfig(tol=1e-8))
    out["fgmres_soc_x"] = xs2
    out["fgmres_soc_iters"] = np.array(rep2.iterations)
    out["fgmres_soc_hist"] = rep2.residual_history
    out["rhs_packed"] = rhs
    np.savez_compressed(OUT / f"{name}.npz", **out)


def gen_basis_fem():
    basis, bench, fem, krylov, ops, pre, problems, rf = _ref()
    out = {}
    mi = basis.enumerate_multi_indices(3, 3)
    out["mi_3_3"] = mi.as_array()
    out["levels_3_3"] = np.array(basis.level_partition(mi).boundaries)
    mi4 = basis.enumerate_multi_indices(4, 2)
    out["mi_4_2"] = mi4.as_array()
    coeff = basis.enumerate_multi_indices(3, 2)
    tp = basis.build_triple_products(mi, coeff, gamma=1.0)
    out["n_H"] = np.array(len(tp.matrices))
    for t, h in enumerate(tp.matrices):
        csr_parts(f"H{t}", h, out)
    out["hermite_table"] = np.array([[[basis.univariate_triple(i, j, k) for k in range(5)] for j in range(5)]
                                     for i in range(5)])
    grid = fem.build_grid(5)
    field = fem.sample_coefficient(grid, lambda x, y: 1.0 + 0.5 * x * y + 0.1 * x)
    csr_parts("mass", fem.assemble_mass(grid), out)
    csr_parts("mass_full", fem.assemble_mass(grid, eliminate_boundary=False), out)
    csr_parts("stiff", fem.assemble_stiffness(grid, field), out)
    out["field"] = field.values
    out["interp"] = fem.interpolate_nodal(grid, lambda x, y: np.sin(x) * np.cos(y))
    out["gauss_x"] = grid.gauss_x
    out["gauss_y"] = grid.gauss_y
    spec = rf.CovarianceSpec(sigma_k=0.4, ell1=0.7, ell2=1.3)
    kl = rf.kl_expand(spec, fem.build_grid(6), 5)
    out["kl_vals"] = kl.eigenvalues
    out["kl_modes"] = np.stack([f.values for f in kl.mode_fields])
    cidx = basis.enumerate_multi_indices(5, 2)
    logn = rf.lognormal_coefficient(kl, cidx)
    out["logn_fields"] = np.stack([f.values for f in logn.coeff_fields])
    np.savez_compressed(OUT / "basis_fem.npz", **out)


def gen_time(name, n, m_xi, p, n_t, beta):
    """Time-dependent all-at-once KKT (operators.py:204-324) and the PINT
    preconditioner (preconditioners.py:198-208, 278-333)."""
    basis, bench, fem, krylov, ops, pre, problems, rf = _ref()
    rng = np.random.default_rng(SEED + 100 + n)
    bundle = problems.build_time_problem(n=n, m_xi=m_xi, p=p, sigma_k=0.3, beta=beta, n_t=n_t,
                                         coefficient="affine")
    sys_ = bundle.system
    st = sys_.steady
    out = {"n": np.array(n), "beta": np.array(beta), "gamma": np.array(st.gamma), "n_t": np.array(n_t),
           "boundaries": np.array(bundle.partition.boundaries, dtype=np.int64), "n_terms": np.array(st.n_terms)}
    csr_parts("M", st.mass, out)
    for t, a in enumerate(st.stiffness):
        csr_parts(f"A{t}", a, out)
    for t, h in enumerate(st.triple.matrices):
        csr_parts(f"H{t}", h, out)
    out["weight_diag"] = st.triple.weight_diagonal
    out["target"] = st.target
    out["y0"] = sys_.initial_state
    size = 3 * sys_.block_size()
    v = rng.standard_normal(size)
    out["v"] = v
    out["kkt"] = ops.time_kkt_apply(sys_, v)
    out["rhs"] = ops.time_rhs(sys_)
    for n_tau in sorted({1, st.n_terms}):
        prec = pre.build_time_preconditioner(sys_, bundle.partition, mass_solver="cheb5", n_tau=n_tau)
        out[f"pint_tau{n_tau}"] = prec.apply(v)
    xs, rep = bench.solve_bundle(bundle, "cheb5", st.n_terms, 1e-6)
    out["fgmres_x"] = xs
    out["fgmres_iters"] = np.array(rep.iterations)
    np.savez_compressed(OUT / f"{name}.npz", **out)


if __name__ == "__main__":
    gen_kron_random()
    gen_basis_fem()
    gen_steady("steady_affine_n6", 6, 2, 2, "affine", None, 0.3, 1e-2)
    gen_steady("steady_logn_n4", 4, 2, 2, "lognormal", 4, 0.3, 1e-2)
    gen_time("time_affine_n6", 6, 2, 2, 4, 1e-2)
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
