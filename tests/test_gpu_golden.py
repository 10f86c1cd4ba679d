"""GPU parity against the reference's golden vectors (tests/golden/*.npz) and
the CPU oracle: every hot-path entry point, through the drop-in Python API
(NumPy in -> C ABI -> sm_100a kernels -> NumPy out).

Tolerances (BASELINE.json north_star): operator / preconditioner outputs
1e-12 relative to max|ref|; Krylov iteration counts +-1; solutions 1e-8."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

from golden_io import csr, load, steady_case

pytestmark = pytest.mark.gpu

CASES = ["steady_affine_n6", "steady_logn_n4"]
OP_TOL = 1e-12


def _close(a, b, tol=OP_TOL):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    b = np.asarray(b)
    scale = float(np.abs(b).max())
    err = float(np.abs(a - b).max()) / scale if scale > 0 else float(np.abs(a).max())
    assert err <= tol, f"relative error {err:.3e} > {tol:.1e}"


def _system(c):
    from paper_2512_23804_b200.basis import LevelPartition, TripleProductSet
    from paper_2512_23804_b200.operators import SteadyKKT

    n_xi = c["x"].shape[1]
    w = c["weight_diag"]
    pen = sp.diags((np.arange(n_xi) > 0).astype(float), format="csr")
    triple = TripleProductSet(matrices=c["couplings"], variance_penalty=pen,
                              objective_weight=sp.diags(w, format="csr"), gamma=float(c["gamma"]))
    sys_ = SteadyKKT(mass=c["mass"], stiffness=c["stiffness"], triple=triple, beta=float(c["beta"]),
                     gamma=float(c["gamma"]), target=c["target"])
    return sys_, LevelPartition(boundaries=c["boundaries"])


def test_kron_random_dense_terms():
    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply, kron_apply_sliced

    g = load("kron_random")
    t = int(g["terms"])
    op = KroneckerSumOperator(couplings=[csr(g, f"H{i}") for i in range(t)],
                              operators=[csr(g, f"A{i}") for i in range(t)])
    _close(kron_apply(op, g["x"]), g["W"])
    _close(kron_apply_sliced(op, g["x"], (1, 4), (2, 5), 3), g["W_sliced_1_4__2_5_t3"])


@pytest.mark.parametrize("name", CASES)
def test_operators(name):
    from paper_2512_23804_b200.operators import kron_apply, kron_apply_sliced, steady_kkt_apply
    from paper_2512_23804_b200.preconditioners import chebyshev_mass_solve

    c = steady_case(name)
    sys_, part = _system(c)
    op = sys_.stiffness_operator()
    _close(kron_apply(op, c["x"]), c["W"])
    n_xi = c["x"].shape[1]
    for lvl, (lo, hi) in enumerate(part.ranges()):
        _close(kron_apply_sliced(op, c["x"], (0, lo), (lo, hi), op.n_terms), c[f"before_{lvl}"])
        _close(kron_apply_sliced(op, c["x"], (hi, n_xi), (lo, hi), op.n_terms), c[f"after_{lvl}"])
    for got, key in zip(steady_kkt_apply(sys_, c["r_y"], c["r_u"], c["r_lam"]), ("kkt_y", "kkt_u", "kkt_lam")):
        _close(got, c[key])
    _close(chebyshev_mass_solve(c["mass"], c["r_y"], 5), c["cheb5"])


@pytest.mark.parametrize("name", CASES)
def test_sweeps(name):
    from paper_2512_23804_b200.preconditioners import (
        build_coupled_preconditioner,
        build_steady_preconditioner,
        build_sweep,
        richardson_hgs,
    )

    c = steady_case(name)
    sys_, part = _system(c)
    for n_tau in sorted({1, 2, c["n_t"]}):
        prec = build_steady_preconditioner(sys_, part, mass_solver="cheb5", n_tau=n_tau)
        _close(prec.sweep.apply(c["r_lam"]), c[f"hgs_tau{n_tau}"])
        _close(richardson_hgs(prec.z_operator, prec.sweep, c["r_lam"], 2), c[f"rich2_tau{n_tau}"])
        for got, key in zip(prec.apply(c["r_y"], c["r_u"], c["r_lam"]), ("bd_y", "bd_u", "bd_lam")):
            _close(got, c[f"{key}_tau{n_tau}"])
        soc = build_coupled_preconditioner(sys_, part, n_tau=n_tau)
        for got, key in zip(soc.apply(c["r_y"], c["r_u"], c["r_lam"]), ("soc_y", "soc_u", "soc_lam")):
            _close(got, c[f"{key}_tau{n_tau}"])
    _, fsweep = build_sweep(c["couplings"][: c["n_t"]], c["stiffness"], part, c["n_t"])
    _close(fsweep.apply(c["x"]), c["fwd_hgs"])


def _device_callables(sys_, prec):
    import torch

    from paper_2512_23804_b200.operators import steady_kkt_apply_device

    n = sys_.block_size()
    shape = (sys_.n_h, sys_.n_xi)

    def split(v):
        return [v[i * n:(i + 1) * n].view(shape) for i in range(3)]

    def apply_op(v):
        out = torch.empty_like(v)
        steady_kkt_apply_device(sys_, *split(v), tuple(split(out)))
        return out

    def apply_prec(v):
        out = torch.empty_like(v)
        prec.apply_device(*split(v), outs=tuple(split(out)))
        return out

    return apply_op, apply_prec


def _packed_rhs_nodemajor(c):
    # golden rhs is packed F-order blocks [vec Y; vec U; vec L]; convert to node-major blocks
    n_h, n_xi = c["x"].shape
    size = n_h * n_xi
    blocks = [c["rhs_packed"][i * size:(i + 1) * size].reshape((n_h, n_xi), order="F") for i in range(3)]
    return np.concatenate([np.ascontiguousarray(b).ravel() for b in blocks])


def _to_fpacked(x, shape):
    n_h, n_xi = shape
    size = n_h * n_xi
    return np.concatenate([x[i * size:(i + 1) * size].reshape(shape).reshape(-1, order="F") for i in range(3)])


@pytest.mark.parametrize("name", CASES)
def test_fgmres_end_to_end(name):
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, fgmres
    from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, build_steady_preconditioner

    c = steady_case(name)
    sys_, part = _system(c)
    b = torch.as_tensor(_packed_rhs_nodemajor(c)).cuda()
    shape = c["x"].shape
    for kind, key in (("bd", "fgmres_bd"), ("soc", "fgmres_soc")):
        prec = (build_steady_preconditioner(sys_, part, "cheb5", c["n_t"]) if kind == "bd"
                else build_coupled_preconditioner(sys_, part))
        op, pr = _device_callables(sys_, prec)
        x, rep = fgmres(op, pr, b, FgmresConfig(tol=1e-8))
        assert rep.converged
        assert abs(rep.iterations - int(c[f"{key}_iters"])) <= 1
        xf = _to_fpacked(x.cpu().numpy(), shape)
        ref = c[f"{key}_x"]
        assert np.linalg.norm(xf - ref) <= 1e-8 * np.linalg.norm(ref)


def test_device_and_numpy_paths_agree(rng):
    import torch

    from paper_2512_23804_b200.operators import kron_apply

    c = steady_case("steady_affine_n6")
    sys_, _ = _system(c)
    op = sys_.stiffness_operator()
    x = rng.standard_normal(c["x"].shape)
    a = kron_apply(op, x)
    d = kron_apply(op, torch.as_tensor(x).cuda())
    assert d.is_cuda
    assert np.array_equal(a, d.cpu().numpy())
    xf = np.asfortranarray(x)
    assert np.array_equal(kron_apply(op, xf), a)


def test_shape_errors():
    from paper_2512_23804_b200.operators import kron_apply, kron_apply_sliced

    c = steady_case("steady_affine_n6")
    sys_, _ = _system(c)
    op = sys_.stiffness_operator()
    with pytest.raises(ValueError):
        kron_apply(op, np.zeros((3, 3)))
    with pytest.raises(ValueError):
        kron_apply_sliced(op, c["x"], (0, 99), (0, 1), 1)
    with pytest.raises(ValueError):
        kron_apply_sliced(op, c["x"], (0, 1), (0, 1), 0)
