"""Preconditioners on the B200: drop-in for `sgkkt.preconditioners`
(reference pkg/src/sgkkt/preconditioners.py).

* hGS  — ``HierarchicalGaussSeidel`` (paper Alg. 1; reference :113-165):
  symmetric block Gauss-Seidel over degree levels.  Per level one fused
  coupling launch (rhs = r[:, lvl] - sum_{1<=t<n_tau} A_t V[:, src] H_t[src, lvl])
  writes the right-hand side in place, then the level's columns are solved
  together by the GPU triangular solves on the host-computed lead factor.
* hGSoc — ``CoupledSweepPreconditioner`` (paper Algs. 2-3; reference
  :336-434): same sweep on the coupled (y, u, lambda) system; one launch
  builds all three level right-hand sides, one P~ solve on the 3-segment
  stack.
* ``SteadyKKTPreconditioner`` (reference :227-255) with Chebyshev mass
  solves (:70-98) and the Richardson-wrapped hGS Schur approximation
  (:172-184) — SPD, the MINRES-admissible choice.

All sweeps run on one stream without host synchronisation.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import scipy.sparse as sp
import torch
from scipy.sparse import csr_matrix

from . import _lib
from .basis import LevelPartition
from .device import DevicePattern, DeviceProgram, as_device_state, run_program
from .fastdiag import fastdiag_factor, fastdiag_kkt_factor
from .linalg import LUFactors, sparse_lu
from .operators import KroneckerSumOperator, SteadyKKT, _finish, kron_apply
from .program import compile_program, coupling_from_csr
from .vec import axpby, colscale

__all__ = [
    "CHEB_LAMBDA_MAX",
    "CHEB_LAMBDA_MIN",
    "ChebyshevConfig",
    "CoupledSweepPreconditioner",
    "LEAD_SOLVERS",
    "HierarchicalGaussSeidel",
    "SteadyKKTPreconditioner",
    "build_coupled_preconditioner",
    "build_steady_preconditioner",
    "build_sweep",
    "chebyshev_mass_solve",
    "deterministic_kkt_matrix",
    "hgs_apply",
    "make_mass_solver",
    "richardson_hgs",
    "shifted_lead_terms",
]

CHEB_LAMBDA_MIN = 0.25
CHEB_LAMBDA_MAX = 2.25
_CHEB_ALPHA = 0.5 * (CHEB_LAMBDA_MIN + CHEB_LAMBDA_MAX)
_CHEB_RHO = (CHEB_LAMBDA_MAX - CHEB_LAMBDA_MIN) / (CHEB_LAMBDA_MAX + CHEB_LAMBDA_MIN)


@dataclass(frozen=True)
class ChebyshevConfig:
    its: int = 5

    def __post_init__(self):
        if self.its < 1:
            raise ValueError("need at least one Chebyshev step")


def _cheb_omegas(its: int) -> list[float]:
    """Relaxation sequence of the reference code (preconditioners.py:89-97):
    1, 1/(1-rho^2/2), then 1/(1-omega rho^2/4)."""
    out = []
    omega = 1.0
    for k in range(its):
        if k == 1:
            omega = 1.0 / (1.0 - _CHEB_RHO**2 / 2.0)
        elif k > 1:
            omega = 1.0 / (1.0 - omega * _CHEB_RHO**2 / 4.0)
        out.append(omega)
    return out


class _DeviceMass:
    """Mass matrix on a device pattern slice + the Chebyshev diagonal scale."""

    def __init__(self, mass: csr_matrix, pattern: DevicePattern | None = None, slice_: int = 0):
        diag = mass.diagonal()
        if np.any(diag == 0.0):
            raise ValueError("mass matrix has a zero diagonal entry")
        self.mass = mass
        self.pattern = pattern if pattern is not None else DevicePattern([mass])
        self.slice = slice_ if pattern is not None else 0
        self.scale = torch.as_tensor(1.0 / (_CHEB_ALPHA * diag)).to(self.pattern._vals.device)

    def cheb(self, b: torch.Tensor, its: int) -> torch.Tensor:
        b2 = b.reshape(b.shape[0], -1)
        return self._run(b2, 1, b2.shape[1], its).reshape(b.shape)

    def cheb_batched(self, b: torch.Tensor, its: int) -> torch.Tensor:
        """chebyshev_mass_solve on each (N, n_cols) block of a (n_b, N, n_cols)
        stack in one launch per step (the time steps of the PINT
        preconditioner); each block's result equals `cheb` on it bitwise."""
        if b.dim() != 3:
            raise ValueError("expected a (n_blocks, N, n_cols) stack")
        return self._run(b, b.shape[0], b.shape[2], its)

    def _run(self, b2: torch.Tensor, n_batch: int, n_cols: int, its: int) -> torch.Tensor:
        if not b2.is_contiguous():
            b2 = b2.contiguous()
        # x0 = x_{-1} = 0: passed as NULL (the kernel reads no zero buffers)
        x_prev = x = None
        lib = _lib.lib()
        stream = _lib.stream_ptr()
        for omega in _cheb_omegas(its):
            x_new = torch.empty_like(b2)
            rc = lib.sgk_cheb_step_batched(
                self.pattern.struct, self.slice, self.scale.data_ptr(), n_batch, n_cols, b2.data_ptr(),
                None if x is None else x.data_ptr(), None if x_prev is None else x_prev.data_ptr(),
                x_new.data_ptr(), omega, stream,
            )
            _lib.check(rc, "sgk_cheb_step")
            x_prev, x = x, x_new
        if x is None:  # its == 0
            x = torch.zeros_like(b2)
        return x


# device copies of mass matrices used by chebyshev_mass_solve, keyed by the
# matrix object; an entry (and its device buffers) is dropped when the matrix
# is garbage-collected
_MASS_CACHE: dict[int, tuple[weakref.ref, _DeviceMass]] = {}


def _device_mass(mass: csr_matrix) -> _DeviceMass:
    key = id(mass)
    hit = _MASS_CACHE.get(key)
    if hit is None or hit[0]() is not mass:
        hit = (weakref.ref(mass), _DeviceMass(mass))
        _MASS_CACHE[key] = hit
        weakref.finalize(mass, _MASS_CACHE.pop, key, None)
    return hit[1]


def chebyshev_mass_solve(mass: csr_matrix, b, cfg: ChebyshevConfig | int = 5):
    """Chebyshev semi-iteration for M x = b, all columns at once
    (reference preconditioners.py:70-98)."""
    its = cfg.its if isinstance(cfg, ChebyshevConfig) else int(cfg)
    if its < 1:
        raise ValueError("need at least one Chebyshev step")
    dm = _device_mass(mass)
    bd, host = as_device_state(b)
    if bd.shape[0] != mass.shape[0]:
        raise ValueError("right-hand side length does not match the mass matrix")
    return _finish(dm.cheb(bd, its), host, b)


def make_mass_solver(mass: csr_matrix, kind: str, pattern: DevicePattern | None = None, slice_: int = 0):
    """'cheb5' / 'cheb10' / 'direct' mass-block solver (reference :101-110)."""
    if kind == "direct":
        factor = sparse_lu(mass)
        return factor.solve
    if kind.startswith("cheb"):
        its = ChebyshevConfig(its=int(kind[4:])).its
        dm = _DeviceMass(mass, pattern, slice_) if pattern is not None else _device_mass(mass)

        def solve(b):
            bd, host = as_device_state(b)
            return _finish(dm.cheb(bd, its), host, b)

        solve.device_mass = dm
        solve.its = its
        return solve
    raise ValueError(f"unknown mass solver {kind!r}")


@dataclass(frozen=True, eq=False)
class HierarchicalGaussSeidel:
    """Symmetric block Gauss-Seidel sweep over degree levels
    (reference preconditioners.py:113-165; paper Alg. 1)."""

    operator: KroneckerSumOperator
    partition: LevelPartition
    n_tau: int
    lead_factor: LUFactors
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if not 1 <= self.n_tau <= self.operator.n_terms:
            raise ValueError("n_tau out of range")

    def _programs(self):
        progs = self._cache.get("progs")
        if progs is None:
            n_xi = self.operator.shape[1]
            ranges = self.partition.ranges()
            fwd = []
            for lo, hi in ranges:
                # coupling to earlier levels only; the first term (identity) has
                # no cross-level entries (reference :139-140)
                fwd.append(self.operator.program([(0, lo)], (lo, hi), 1, self.n_tau, -1.0))
            bwd = []
            for lo, hi in reversed(ranges[:-1]):
                bwd.append(self.operator.program([(0, lo), (hi, n_xi)], (lo, hi), 1, self.n_tau, -1.0))
            progs = (fwd, bwd)
            self._cache["progs"] = progs
        return progs

    def apply_device(self, r: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        n_h, n_xi = self.operator.shape
        v = out if out is not None else torch.empty((n_h, n_xi), dtype=torch.float64, device=r.device)
        fwd, bwd = self._programs()
        pat = self.operator.pattern
        fac = self.lead_factor.device_factors
        ranges = self.partition.ranges()
        for (lo, hi), prog in zip(ranges, fwd):
            run_program(pat, prog, [(v, 0)], [(v, lo)], [(r, lo)], alpha=[1.0], beta=[1.0])
            fac.solve_segments([(v, lo)], [(v, lo)], hi - lo)
        for (lo, hi), prog in zip(reversed(ranges[:-1]), bwd):
            run_program(pat, prog, [(v, 0)], [(v, lo)], [(r, lo)], alpha=[1.0], beta=[1.0])
            fac.solve_segments([(v, lo)], [(v, lo)], hi - lo)
        return v

    def apply(self, r):
        n_h, n_xi = self.operator.shape
        if tuple(r.shape) != (n_h, n_xi):
            raise ValueError(f"residual shape {tuple(r.shape)} does not match {self.operator.shape}")
        rd, host = as_device_state(r, (n_h, n_xi))
        return _finish(self.apply_device(rd), host, r)


def hgs_apply(sweep: HierarchicalGaussSeidel, r):
    return sweep.apply(r)


def _richardson_device(op: KroneckerSumOperator, sweep, b: torch.Tensor, n_steps: int) -> torch.Tensor:
    x = sweep.apply_device(b) if hasattr(sweep, "apply_device") else as_device_state(sweep.apply(b))[0]
    n_xi = op.shape[1]
    for _ in range(n_steps - 1):
        # x + sweep(b - Z x): residual fused into one program launch (init=b, alpha=-1)
        res = torch.empty_like(b)
        prog = op.program([(0, n_xi)], (0, n_xi), 0, op.n_terms)
        run_program(op.pattern, prog, [(x, 0)], [(res, 0)], [(b, 0)], alpha=[-1.0], beta=[1.0])
        corr = sweep.apply_device(res) if hasattr(sweep, "apply_device") else as_device_state(sweep.apply(res))[0]
        axpby(x, corr, 1.0, 1.0)
    return x


def richardson_hgs(op: KroneckerSumOperator, sweep, b, n_steps: int = 1):
    """Richardson from zero preconditioned by the sweep (reference :172-184)."""
    if n_steps < 1:
        raise ValueError("need at least one Richardson step")
    bd, host = as_device_state(b, op.shape)
    return _finish(_richardson_device(op, sweep, bd, n_steps), host, b)


def shifted_lead_terms(sys: SteadyKKT) -> list[csr_matrix]:
    """[A_1 + sqrt((1+gamma)/beta) M, A_2, ...] (reference :187-195)."""
    shift = np.sqrt((1.0 + sys.gamma) / sys.beta)
    lead = (sys.stiffness[0] + shift * sys.mass).tocsr()
    return [lead] + [a.tocsr() for a in sys.stiffness[1:]]


LEAD_SOLVERS = ("lu", "lu_nd", "lu_tp", "fastdiag")
TP_THRESHOLD = 0.01  # "lu_tp": SuperLU threshold partial pivoting


def _lead_factor(lead, mass, lead_solver: str):
    """The lead-term factor: the reference's SuperLU ("lu", default; GPU
    triangular solves), SuperLU on a nested-dissection ordering of the grid
    ("lu_nd": same solve, shallower triangles), SuperLU with threshold partial
    pivoting ("lu_tp", pivot threshold 0.01), or the depth-free fast
    diagonalisation of a Kronecker-sum lead ("fastdiag", SURVEY §8(f) row 3;
    needs the mass matrix, raises ValueError when the lead is not a Kronecker
    sum)."""
    if lead_solver == "lu":
        return sparse_lu(lead)
    if lead_solver == "lu_nd":
        return sparse_lu(lead, ordering="nd")
    if lead_solver == "lu_tp":
        return sparse_lu(lead, pivot_threshold=TP_THRESHOLD)
    if lead_solver == "fastdiag":
        if mass is None:
            raise ValueError("lead_solver='fastdiag' needs the mass matrix")
        return fastdiag_factor(lead, mass)
    raise ValueError(f"unknown lead solver {lead_solver!r} (expected one of {LEAD_SOLVERS})")


def build_sweep(couplings, terms, partition: LevelPartition, n_tau: int, *, lead_solver: str = "lu",
                mass=None):
    """Kronecker operator + sweep with a host-factored lead term
    (reference :211-224).  With unshifted stiffness terms this is the hGS
    preconditioner of the forward problem (configs 1 and 3)."""
    op = KroneckerSumOperator(couplings=list(couplings), operators=list(terms))
    sweep = HierarchicalGaussSeidel(operator=op, partition=partition, n_tau=n_tau,
                                    lead_factor=_lead_factor(terms[0], mass, lead_solver))
    return op, sweep


_build_sweep = build_sweep


@dataclass(frozen=True, eq=False)
class SteadyKKTPreconditioner:
    """Block-diagonal Benner-type preconditioner (reference :227-255):
    diag( M_gamma^-1 (Chebyshev), (beta M)^-1 (Chebyshev), Z^-1 M_gamma Z^-1 (hGS) )."""

    system: SteadyKKT
    mass_solve: Callable
    z_operator: KroneckerSumOperator
    sweep: HierarchicalGaussSeidel
    richardson_steps: int = 1
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def _weighted_mass_program(self) -> DeviceProgram:
        prog = self._cache.get("wm")
        if prog is None:
            sys = self.system
            n_xi = sys.n_xi
            w = sys.triple.objective_weight.tocsr()
            cp = coupling_from_csr(0, 0, sys.mass_slice, w, (0, n_xi), (0, n_xi), 1.0)
            prog = DeviceProgram([cp], (n_xi,), n_inputs=1)
            self._cache["wm"] = prog
        return prog

    def _weights(self) -> torch.Tensor:
        w = self._cache.get("w")
        if w is None:
            w = torch.as_tensor(self.system.triple.weight_diagonal.astype(np.float64)).cuda()
            self._cache["w"] = w
        return w

    def _mass_dev(self, b: torch.Tensor) -> torch.Tensor:
        out = self.mass_solve(b)
        return out if isinstance(out, torch.Tensor) and out.is_cuda else as_device_state(out)[0]

    def schur_apply_device(self, r_lam: torch.Tensor) -> torch.Tensor:
        z1 = _richardson_device(self.z_operator, self.sweep, r_lam, self.richardson_steps)
        wz = torch.empty_like(z1)
        run_program(self.system.pattern, self._weighted_mass_program(), [(z1, 0)], [(wz, 0)],
                    alpha=[1.0], beta=[0.0])
        return _richardson_device(self.z_operator, self.sweep, wz, self.richardson_steps)

    def schur_apply(self, r_lam):
        rd, host = as_device_state(r_lam, (self.system.n_h, self.system.n_xi))
        return _finish(self.schur_apply_device(rd), host, r_lam)

    def apply_device(self, r_y, r_u, r_lam, outs=None):
        sys = self.system
        n_h, n_xi = sys.n_h, sys.n_xi
        outs = outs or tuple(torch.empty((n_h, n_xi), dtype=torch.float64, device=r_y.device) for _ in range(3))
        colscale(self._mass_dev(r_y), self._weights(), 1.0, outs[0], invert=True)
        colscale(self._mass_dev(r_u), None, 1.0 / sys.beta, outs[1])
        outs[2].copy_(self.schur_apply_device(r_lam))
        return outs

    def apply(self, r_y, r_u, r_lam):
        shape = (self.system.n_h, self.system.n_xi)
        ds = []
        host = False
        for blk in (r_y, r_u, r_lam):
            d, h = as_device_state(blk, shape)
            ds.append(d)
            host = host or h
        outs = self.apply_device(*ds)
        return tuple(_finish(o, host, r_y) for o in outs)


def build_steady_preconditioner(sys: SteadyKKT, partition: LevelPartition, mass_solver: str = "cheb5",
                                n_tau: int | None = None, richardson_steps: int = 1, *,
                                lead_solver: str = "lu") -> SteadyKKTPreconditioner:
    n_tau = sys.n_terms if n_tau is None else n_tau
    z_op, sweep = build_sweep(sys.triple.matrices[: sys.n_terms], shifted_lead_terms(sys), partition, n_tau,
                              lead_solver=lead_solver, mass=sys.mass)
    if mass_solver.startswith("cheb"):
        ms = make_mass_solver(sys.mass, mass_solver, sys.pattern, sys.mass_slice)
    else:
        ms = make_mass_solver(sys.mass, mass_solver)
    return SteadyKKTPreconditioner(system=sys, mass_solve=ms, z_operator=z_op, sweep=sweep,
                                   richardson_steps=richardson_steps)


@dataclass(frozen=True, eq=False)
class CoupledSweepPreconditioner:
    """hGSoc: hierarchical sweep over the coupled KKT system
    (reference preconditioners.py:336-434; paper Algs. 2-3)."""

    system: SteadyKKT
    partition: LevelPartition
    n_tau: int
    kkt_factor: LUFactors
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def _level_program(self, src_ranges, dst) -> DeviceProgram:
        sys = self.system
        m = sys.mass_slice
        weight = sys.triple.objective_weight.tocsr()
        ident = sys.triple.matrices[0].tocsr()
        cps = []
        # inputs 0=v_y, 1=v_u, 2=v_lam ; outputs 0=rhs_y, 1=rhs_u, 2=rhs_lam
        # (reference _level_rhs :386-409; mass couplings vanish for diagonal H
        #  but are consulted, :348-351)
        for src in src_ranges:
            cps.append(coupling_from_csr(0, 0, m, weight, src, dst, -1.0))
            for t in range(self.n_tau):
                h = sys.triple.matrices[t].tocsr()
                cps.append(coupling_from_csr(2, 0, t, h, src, dst, 1.0))
                cps.append(coupling_from_csr(0, 2, t, h, src, dst, 1.0))
            cps.append(coupling_from_csr(1, 1, m, ident, src, dst, -sys.beta))
            cps.append(coupling_from_csr(2, 1, m, ident, src, dst, -1.0))
            cps.append(coupling_from_csr(1, 2, m, ident, src, dst, -1.0))
        w = dst[1] - dst[0]
        return DeviceProgram(cps, (w, w, w), n_inputs=3)

    def _programs(self):
        progs = self._cache.get("progs")
        if progs is None:
            n_xi = self.system.n_xi
            ranges = self.partition.ranges()
            fwd = [self._level_program([(0, lo)], (lo, hi)) for lo, hi in ranges]
            bwd = [self._level_program([(0, lo), (hi, n_xi)], (lo, hi)) for lo, hi in reversed(ranges[:-1])]
            progs = (fwd, bwd)
            self._cache["progs"] = progs
        return progs

    def apply_device(self, r_y, r_u, r_lam, outs=None):
        sys = self.system
        n_h, n_xi = sys.n_h, sys.n_xi
        outs = outs or tuple(torch.empty((n_h, n_xi), dtype=torch.float64, device=r_y.device) for _ in range(3))
        vy, vu, vl = outs
        fwd, bwd = self._programs()
        pat = sys.pattern
        fac = self.kkt_factor.device_factors
        ranges = self.partition.ranges()

        def level(prog, lo, hi):
            run_program(pat, prog, [(vy, 0), (vu, 0), (vl, 0)], [(vy, lo), (vu, lo), (vl, lo)],
                        [(r_y, lo), (r_u, lo), (r_lam, lo)], alpha=[1.0] * 3, beta=[1.0] * 3)
            segs = [(vy, lo), (vu, lo), (vl, lo)]
            fac.solve_segments(segs, segs, hi - lo)

        for (lo, hi), prog in zip(ranges, fwd):
            level(prog, lo, hi)
        for (lo, hi), prog in zip(reversed(ranges[:-1]), bwd):
            level(prog, lo, hi)
        return outs

    def apply(self, r_y, r_u, r_lam):
        shape = (self.system.n_h, self.system.n_xi)
        ds = []
        host = False
        for blk in (r_y, r_u, r_lam):
            d, h = as_device_state(blk, shape)
            ds.append(d)
            host = host or h
        outs = self.apply_device(*ds)
        return tuple(_finish(o, host, r_y) for o in outs)


def deterministic_kkt_matrix(sys: SteadyKKT) -> csr_matrix:
    """P~ = [M 0 -A_1; 0 beta M M; -A_1 M 0] (reference :437-448)."""
    m = sys.mass
    a1 = sys.stiffness[0]
    return sp.bmat([[m, None, -a1], [None, sys.beta * m, m], [-a1, m, None]], format="csr")


def build_coupled_preconditioner(sys: SteadyKKT, partition: LevelPartition,
                                 n_tau: int | None = None, *, lead_solver: str = "lu") -> CoupledSweepPreconditioner:
    """hGSoc with the P~ factor from SuperLU ("lu", the reference's
    preconditioners.py:451-462) or the fast diagonalisation ("fastdiag")."""
    n_tau = sys.n_terms if n_tau is None else n_tau
    if not 1 <= n_tau <= sys.n_terms:
        raise ValueError("n_tau out of range")
    if lead_solver in ("lu", "lu_nd"):
        # the indefinite P~ pivots: a nested-dissection order does not survive
        # partial pivoting (config 5: depth 4.3k -> 44k), so P~ keeps COLAMD
        factor = sparse_lu(deterministic_kkt_matrix(sys))
    elif lead_solver == "lu_tp":
        # threshold pivoting keeps more diagonal pivots: shallower, sparser
        # triangles (config 5: chain-group depth 218 -> 146)
        factor = sparse_lu(deterministic_kkt_matrix(sys), pivot_threshold=TP_THRESHOLD)
    elif lead_solver == "fastdiag":
        factor = fastdiag_kkt_factor(sys.stiffness[0], sys.mass, sys.beta)
    else:
        raise ValueError(f"unknown lead solver {lead_solver!r} (expected one of {LEAD_SOLVERS})")
    return CoupledSweepPreconditioner(system=sys, partition=partition, n_tau=n_tau, kkt_factor=factor)
