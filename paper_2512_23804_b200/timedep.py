"""Time-dependent all-at-once KKT operator and the parallel-in-time (PINT)
preconditioner on the B200 — SURVEY §8(f) row 1, a batched reuse of the
steady kernels over N_t implicit-Euler steps.

Reference: operators.py:204-324 (TimeStencil, build_time_stencil, TimeKKT,
split/join_time_blocks, time_kkt_apply, time_rhs) and preconditioners.py:
198-208, 278-333 (time_lead_terms, TimeKKTPreconditioner,
build_time_preconditioner); paper Alg. 4.

Layouts.  The reference packs an all-at-once vector as [y steps; u steps;
lambda steps], each step an F-order vec of an (N, n_xi) block.  On the device
the same vector is (3, N_t, N, n_xi) node-major blocks; NumPy inputs are
converted at the boundary (`to_device_layout` / `from_device_layout`).

The operator (`time_kkt_apply`) is ONE fused program launch over the shared
pattern on interleaved step columns (column l*N_t + k = step k's column l):
the steady KKT couplings with each step's tau / trapezoid-weight factors as
diagonal N_t x N_t factors, and the time couplings M lambda_{k+1} and
M y_{k-1} as column shifts; a transpose per block on each side.
`time_kkt_apply_device` keeps the per-step form (one program per step plus
one launch for the time couplings).  The PINT preconditioner is block diagonal in
time: every step runs the Chebyshev mass solves and the Richardson-wrapped
hGS sweep with the time-shifted lead term (1 + tau sqrt((1+gamma)/beta)) M +
tau A_1, independently of the other steps (the step order never matters —
reference tests/test_preconditioners.py:339-345).  So the device path runs
all steps at once: the 2 N_t mass solves as one batched Chebyshev launch per
step, and the N_t Schur blocks as ONE sweep over an (N, n_xi*N_t) matrix with
interleaved step columns (couplings H_t (x) I_{N_t}); `step_order=` keeps the
reference's per-step loop.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np
import scipy.sparse as sp
import torch
from scipy.sparse import csr_matrix

from .basis import LevelPartition
from .device import DeviceProgram, as_device_state, device, run_program
from .linalg import csr_from_coo
from .operators import KroneckerSumOperator, SteadyKKT
from .preconditioners import HierarchicalGaussSeidel, _richardson_device, build_sweep, make_mass_solver
from .program import coupling_from_csr
from .vec import colscale, colscale_batched

__all__ = [
    "TimeKKT",
    "TimeKKTPreconditioner",
    "TimeStencil",
    "build_time_preconditioner",
    "build_time_stencil",
    "from_device_layout",
    "join_time_blocks",
    "split_time_blocks",
    "time_kkt_apply",
    "time_kkt_apply_device",
    "time_kkt_apply_interleaved",
    "time_lead_terms",
    "time_rhs",
    "to_device_layout",
]


@dataclass(frozen=True)
class TimeStencil:
    """Implicit-Euler coupling (-1 on the first subdiagonal) and trapezoid
    weights on [0, 1] (reference operators.py:204-223)."""

    n_t: int
    tau: float
    coupling: csr_matrix
    weights: np.ndarray


def build_time_stencil(n_t: int) -> TimeStencil:
    if n_t < 1:
        raise ValueError("need at least one time step")
    idx = np.arange(1, n_t)
    coupling = csr_from_coo(n_t, n_t, idx, idx - 1, -np.ones(n_t - 1))
    w = np.ones(n_t)
    w[0] = 0.5
    w[-1] = 0.5
    return TimeStencil(n_t=n_t, tau=1.0 / n_t, coupling=coupling, weights=w)


@dataclass(frozen=True, eq=False)
class TimeKKT:
    """All-at-once KKT operator of the time-dependent control problem
    (reference operators.py:226-247)."""

    steady: SteadyKKT
    stencil: TimeStencil
    initial_state: np.ndarray
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if np.asarray(self.initial_state).shape != (self.steady.n_h, self.steady.n_xi):
            raise ValueError("initial state shape does not match the system")

    @property
    def n_t(self) -> int:
        return self.stencil.n_t

    @property
    def tau(self) -> float:
        return self.stencil.tau

    def block_size(self) -> int:
        return self.n_t * self.steady.block_size()

    # -- device programs -----------------------------------------------------
    def _step_program(self, wk: float) -> DeviceProgram:
        key = ("step", wk)
        prog = self._cache.get(key)
        if prog is None:
            st = self.steady
            n_xi, T, m = st.n_xi, st.n_terms, st.mass_slice
            tau = self.tau
            full = (0, n_xi)
            wdiag = st.triple.objective_weight.tocsr()
            eye = sp.identity(n_xi, format="csr")
            cps = [coupling_from_csr(0, 0, m, wdiag, full, full, tau * wk)]  # tau w_k (M y) W
            cps.append(coupling_from_csr(2, 0, m, eye, full, full, -1.0))  # - M lam_k
            cps.append(coupling_from_csr(1, 1, m, eye, full, full, st.beta * tau * wk))  # beta tau w_k M u
            cps.append(coupling_from_csr(2, 1, m, eye, full, full, tau))  # tau M lam
            cps.append(coupling_from_csr(0, 2, m, eye, full, full, -1.0))  # - M y_k
            cps.append(coupling_from_csr(1, 2, m, eye, full, full, tau))  # tau M u
            for t in range(T):
                h = st.triple.matrices[t].tocsr()
                cps.append(coupling_from_csr(2, 0, t, h, full, full, -tau))  # - tau A lam
                cps.append(coupling_from_csr(0, 2, t, h, full, full, -tau))  # - tau A y
            prog = DeviceProgram(cps, (n_xi, n_xi, n_xi), n_inputs=3)
            self._cache[key] = prog
        return prog

    def _coupling_program(self, nxt: bool, prv: bool) -> DeviceProgram:
        key = ("couple", nxt, prv)
        prog = self._cache.get(key)
        if prog is None:
            st = self.steady
            n_xi, m = st.n_xi, st.mass_slice
            eye = sp.identity(n_xi, format="csr")
            full = (0, n_xi)
            cps, widths, s = [], [], 0
            if nxt:  # r_y += M lam_{k+1}
                cps.append(coupling_from_csr(s, len(widths), m, eye, full, full, 1.0))
                widths.append(n_xi)
                s += 1
            if prv:  # r_lam += M y_{k-1}
                cps.append(coupling_from_csr(s, len(widths), m, eye, full, full, 1.0))
                widths.append(n_xi)
                s += 1
            prog = DeviceProgram(cps, tuple(widths), n_inputs=s)
            self._cache[key] = prog
        return prog


def _blocks(sys: TimeKKT, v: torch.Tensor):
    """(3, n_t) grid of (N, n_xi) views of a device-layout vector."""
    st = sys.steady
    g = v.view(3, sys.n_t, st.n_h, st.n_xi)
    return g


def _interleaved_kkt_program(sys: TimeKKT) -> DeviceProgram:
    """The whole all-at-once operator as ONE coupling program on interleaved
    step columns (column l*N_t + k = step k's chaos column l): the step
    factors become diagonal N_t x N_t factors of each coupling, and the time
    couplings M lambda_{k+1} -> r_y,k and M y_{k-1} -> r_lam,k become shifts
    in the column space (reference operators.py:284-309)."""
    prog = sys._cache.get("interleaved")
    if prog is None:
        st = sys.steady
        n_xi, T, m, n_t, tau = st.n_xi, st.n_terms, st.mass_slice, sys.n_t, sys.tau
        w = np.asarray(sys.stencil.weights, np.float64)
        kr = lambda a, b: sp.kron(a, b, format="csr")
        ix, it = sp.identity(n_xi, format="csr"), sp.identity(n_t, format="csr")
        nxt = sp.diags(np.ones(n_t - 1), -1, shape=(n_t, n_t), format="csr")  # src step k+1 -> dst step k
        prv = sp.diags(np.ones(n_t - 1), 1, shape=(n_t, n_t), format="csr")  # src step k-1 -> dst step k
        full = (0, n_xi * n_t)
        cps = [coupling_from_csr(0, 0, m, kr(st.triple.objective_weight.tocsr(), sp.diags(tau * w)), full, full, 1.0),
               coupling_from_csr(2, 0, m, kr(ix, nxt - it), full, full, 1.0),  # M (lam_{k+1} - lam_k)
               coupling_from_csr(1, 1, m, kr(ix, sp.diags(st.beta * tau * w)), full, full, 1.0),
               coupling_from_csr(2, 1, m, kr(ix, it), full, full, tau),
               coupling_from_csr(0, 2, m, kr(ix, prv - it), full, full, 1.0),  # M (y_{k-1} - y_k)
               coupling_from_csr(1, 2, m, kr(ix, it), full, full, tau)]
        for t in range(T):
            h = kr(st.triple.matrices[t].tocsr(), it)
            cps.append(coupling_from_csr(2, 0, t, h, full, full, -tau))
            cps.append(coupling_from_csr(0, 2, t, h, full, full, -tau))
        prog = DeviceProgram(cps, (n_xi * n_t,) * 3, n_inputs=3)
        sys._cache["interleaved"] = prog
    return prog


def time_kkt_apply_interleaved(sys: TimeKKT, v: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """time_kkt_apply_device as one program launch between two transposes
    per block ((N_t, N*n_xi) <-> (N*n_xi, N_t)); same operator, the gather
    may sum in a different order than the per-step launches."""
    from . import _lib

    st = sys.steady
    n_t, cells = sys.n_t, st.n_h * st.n_xi
    lib = _lib.lib()
    vi = torch.empty((3, st.n_h, st.n_xi * n_t), dtype=torch.float64, device=v.device)
    oi = torch.empty_like(vi)
    vb = v.view(3, n_t, cells)
    ob = out.view(3, n_t, cells)
    for b in range(3):
        _lib.check(lib.sgk_n2f(n_t, cells, vb[b].data_ptr(), vi[b].data_ptr(), _lib.stream_ptr()), "sgk_n2f")
    run_program(st.pattern, _interleaved_kkt_program(sys), [(vi[0], 0), (vi[1], 0), (vi[2], 0)],
                [(oi[0], 0), (oi[1], 0), (oi[2], 0)], alpha=[1.0] * 3, beta=[0.0] * 3)
    for b in range(3):
        _lib.check(lib.sgk_n2f(cells, n_t, oi[b].data_ptr(), ob[b].data_ptr(), _lib.stream_ptr()), "sgk_n2f")
    return out


def time_kkt_apply_device(sys: TimeKKT, v: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    g = _blocks(sys, v)
    o = _blocks(sys, out)
    pat = sys.steady.pattern
    w = sys.stencil.weights
    for k in range(sys.n_t):
        run_program(pat, sys._step_program(float(w[k])), [(g[0, k], 0), (g[1, k], 0), (g[2, k], 0)],
                    [(o[0, k], 0), (o[1, k], 0), (o[2, k], 0)], alpha=[1.0] * 3, beta=[0.0] * 3)
        nxt, prv = k + 1 < sys.n_t, k > 0
        if nxt or prv:
            ins, outs = [], []
            if nxt:
                ins.append((g[2, k + 1], 0))
                outs.append((o[0, k], 0))
            if prv:
                ins.append((g[0, k - 1], 0))
                outs.append((o[2, k], 0))
            run_program(pat, sys._coupling_program(nxt, prv), ins, outs, inits=list(outs),
                        alpha=[1.0] * len(outs), beta=[1.0] * len(outs))
    return out


def to_device_layout(sys: TimeKKT, v) -> torch.Tensor:
    """Reference packed vector (F-order step blocks) -> device layout."""
    st = sys.steady
    a = np.asarray(v, dtype=np.float64)
    if a.size != 3 * sys.block_size():
        raise ValueError(f"expected length {3 * sys.block_size()}, got {a.size}")
    blocks = a.reshape(3 * sys.n_t, st.n_xi, st.n_h).transpose(0, 2, 1)
    return torch.as_tensor(np.ascontiguousarray(blocks)).to(device()).reshape(-1)


def from_device_layout(sys: TimeKKT, t: torch.Tensor) -> np.ndarray:
    st = sys.steady
    a = t.detach().cpu().numpy().reshape(3 * sys.n_t, st.n_h, st.n_xi)
    return np.ascontiguousarray(a.transpose(0, 2, 1)).reshape(-1)


def split_time_blocks(sys: TimeKKT, v):
    """(y, u, lam) step arrays of a reference-packed vector (operators.py:250-271)."""
    st = sys.steady
    a = np.asarray(v, dtype=np.float64)
    if a.size != 3 * sys.block_size():
        raise ValueError(f"expected length {3 * sys.block_size()}, got {a.size}")
    steps = a.reshape(3, sys.n_t, st.n_xi, st.n_h).transpose(0, 1, 3, 2)
    return steps[0].copy(), steps[1].copy(), steps[2].copy()


def join_time_blocks(y, u, lam) -> np.ndarray:
    return np.concatenate([np.asarray(b)[k].reshape(-1, order="F") for b in (y, u, lam) for k in range(len(b))])


def time_kkt_apply(sys: TimeKKT, v):
    """All-at-once KKT operator (reference operators.py:284-309).  NumPy
    (reference layout) in -> NumPy out; CUDA tensor (device layout) in ->
    CUDA tensor out."""
    if isinstance(v, torch.Tensor) and v.is_cuda:
        if v.numel() != 3 * sys.block_size():
            raise ValueError("vector length does not match the system")
        return time_kkt_apply_interleaved(sys, v.contiguous(), torch.empty_like(v))
    vd = to_device_layout(sys, v)
    return from_device_layout(sys, time_kkt_apply_interleaved(sys, vd, torch.empty_like(vd)))


def time_rhs(sys: TimeKKT) -> np.ndarray:
    """Packed right-hand side (reference operators.py:312-324) — host setup."""
    st = sys.steady
    tau, w = sys.tau, sys.stencil.weights
    mt = np.asarray(st.mass @ np.asarray(st.target))
    b_y = np.stack([tau * w[k] * mt for k in range(sys.n_t)])
    b_u = np.zeros_like(b_y)
    b_l = np.zeros_like(b_y)
    b_l[0] = np.asarray(st.mass @ np.asarray(sys.initial_state))
    return join_time_blocks(b_y, b_u, b_l)


def time_lead_terms(sys: TimeKKT) -> list[csr_matrix]:
    """[(1 + tau sqrt((1+gamma)/beta)) M + tau A_1, tau A_2, ...]
    (reference preconditioners.py:198-208)."""
    st = sys.steady
    tau = sys.tau
    shift = 1.0 + tau * np.sqrt((1.0 + st.gamma) / st.beta)
    return [(shift * st.mass + tau * st.stiffness[0]).tocsr()] + [(tau * a).tocsr() for a in st.stiffness[1:]]


@dataclass(frozen=True, eq=False)
class TimeKKTPreconditioner:
    """Parallel-in-time block-diagonal preconditioner (reference
    preconditioners.py:278-312; paper Alg. 4)."""

    system: TimeKKT
    mass_solve: Callable
    z_operator: KroneckerSumOperator
    sweep: HierarchicalGaussSeidel
    richardson_steps: int = 1
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def _weighted_mass(self, dk: float) -> DeviceProgram:
        key = ("wm", dk)
        prog = self._cache.get(key)
        if prog is None:
            st = self.system.steady
            n_xi = st.n_xi
            cp = coupling_from_csr(0, 0, st.mass_slice, st.triple.objective_weight.tocsr(), (0, n_xi), (0, n_xi), dk)
            prog = DeviceProgram([cp], (n_xi,), n_inputs=1)
            self._cache[key] = prog
        return prog

    def _weights(self) -> torch.Tensor:
        w = self._cache.get("w")
        if w is None:
            w = torch.as_tensor(self.system.steady.triple.weight_diagonal.astype(np.float64)).to(device())
            self._cache["w"] = w
        return w

    def _mass(self, b: torch.Tensor) -> torch.Tensor:
        out = self.mass_solve(b)
        return out if isinstance(out, torch.Tensor) and out.is_cuda else as_device_state(out)[0]

    def _stepwise_schur(self):
        """The lambda block's Z^-1 M_gamma Z^-1 for all N_t steps at once.

        Step k's (N, n_xi) block becomes columns l*N_t + k of one
        (N, n_xi*N_t) matrix (a transpose of the (N_t, N*n_xi) stack), so the
        steps' hGS sweeps are ONE sweep with couplings H_t (x) I_{N_t} and
        level boundaries scaled by N_t: every level solve and coupling
        launch covers all steps (the same per-column arithmetic as the
        per-step loop; the gather may sum in a different order)."""
        bt = self._cache.get("stepwise")
        if bt is None:
            sys = self.system
            st = sys.steady
            n_t, n_xi = sys.n_t, st.n_xi
            eye = sp.identity(n_t, format="csr")
            op = self.z_operator
            op_x = KroneckerSumOperator(couplings=[sp.kron(h, eye, format="csr") for h in op.couplings],
                                        operators=list(op.operators))
            op_x._cache["pattern"] = op.pattern  # same A_t: share the device values
            part_x = LevelPartition(boundaries=np.asarray(self.sweep.partition.boundaries, np.int64) * n_t)
            sweep_x = HierarchicalGaussSeidel(operator=op_x, partition=part_x, n_tau=self.sweep.n_tau,
                                              lead_factor=self.sweep.lead_factor)
            # weighted mass of step k: dk * M Z H_gamma -> H_gamma (x) diag(d)
            wm = sp.kron(st.triple.objective_weight.tocsr(), sp.diags(np.asarray(sys.stencil.weights, np.float64)),
                         format="csr")
            cp = coupling_from_csr(0, 0, st.mass_slice, wm, (0, n_xi * n_t), (0, n_xi * n_t), 1.0)
            bt = (op_x, sweep_x, DeviceProgram([cp], (n_xi * n_t,), n_inputs=1))
            self._cache["stepwise"] = bt
        return bt

    def _schur_all_steps(self, r_lam: torch.Tensor, o_lam: torch.Tensor) -> None:
        from . import _lib

        sys = self.system
        st = sys.steady
        n_t, n_cells = sys.n_t, st.n_h * st.n_xi
        op_x, sweep_x, wm = self._stepwise_schur()
        lib = _lib.lib()
        zin = torch.empty((st.n_h, st.n_xi * n_t), dtype=torch.float64, device=r_lam.device)
        # (N_t, N*n_xi) row-major -> (N*n_xi, N_t): column l*N_t + k of zin is step k's column l
        _lib.check(lib.sgk_n2f(n_t, n_cells, r_lam.data_ptr(), zin.data_ptr(), _lib.stream_ptr()), "sgk_n2f")
        z1 = _richardson_device(op_x, sweep_x, zin, self.richardson_steps)
        ww = torch.empty_like(z1)
        run_program(st.pattern, wm, [(z1, 0)], [(ww, 0)], alpha=[1.0], beta=[0.0])
        z2 = _richardson_device(op_x, sweep_x, ww, self.richardson_steps)
        colscale(z2, None, sys.tau, z2)
        _lib.check(lib.sgk_n2f(n_cells, n_t, z2.data_ptr(), o_lam.data_ptr(), _lib.stream_ptr()), "sgk_n2f")

    def apply_device(self, r: torch.Tensor, out: torch.Tensor, step_order: Sequence[int] | None = None):
        """All steps batched (default), or the per-step loop in `step_order`
        (the reference's structure; block diagonal in time, so any order)."""
        sys = self.system
        st = sys.steady
        tau, wsteps = sys.tau, sys.stencil.weights
        g = _blocks(sys, r)
        o = _blocks(sys, out)
        wv = self._weights()
        batched = step_order is None
        steps = list(range(sys.n_t) if step_order is None else step_order)
        dm = getattr(self.mass_solve, "device_mass", None)
        if dm is not None:
            # the time steps' y and u mass solves are independent: one batched
            # Chebyshev launch per step over all 2 N_t blocks
            its = self.mass_solve.its
            mass_yu = dm.cheb_batched(g[0:2].reshape(2 * sys.n_t, st.n_h, st.n_xi), its).view(
                2, sys.n_t, st.n_h, st.n_xi)
        if batched and dm is not None:
            # y/u column scalings of all steps: one launch each, step scalars on the device
            sc = self._cache.get("step_scales")
            if sc is None:
                sc = torch.tensor([[1.0 / (tau * float(d)) for d in wsteps],
                                   [1.0 / (st.beta * tau * float(d)) for d in wsteps]],
                                  dtype=torch.float64, device=r.device)
                self._cache["step_scales"] = sc
            colscale_batched(mass_yu[0], wv, sc[0], o[0], invert=True)
            colscale_batched(mass_yu[1], None, sc[1], o[1])
            self._schur_all_steps(g[2], o[2])
            return out
        for k in steps:
            dk = float(wsteps[k])
            my = mass_yu[0, k] if dm is not None else self._mass(g[0, k])
            mu = mass_yu[1, k] if dm is not None else self._mass(g[1, k])
            colscale(my, wv, 1.0 / (tau * dk), o[0, k], invert=True)
            colscale(mu, None, 1.0 / (st.beta * tau * dk), o[1, k])
            if batched:
                continue
            z1 = _richardson_device(self.z_operator, self.sweep, g[2, k], self.richardson_steps)
            ww = torch.empty_like(z1)
            run_program(st.pattern, self._weighted_mass(dk), [(z1, 0)], [(ww, 0)], alpha=[1.0], beta=[0.0])
            z2 = _richardson_device(self.z_operator, self.sweep, ww, self.richardson_steps)
            colscale(z2, None, tau, o[2, k])
        if batched:
            self._schur_all_steps(g[2], o[2])
        return out

    def apply(self, r, step_order: Sequence[int] | None = None):
        if isinstance(r, torch.Tensor) and r.is_cuda:
            return self.apply_device(r.contiguous(), torch.empty_like(r), step_order)
        rd = to_device_layout(self.system, r)
        return from_device_layout(self.system, self.apply_device(rd, torch.empty_like(rd), step_order))


def build_time_preconditioner(sys: TimeKKT, partition: LevelPartition, mass_solver: str = "cheb5",
                              n_tau: int | None = None, richardson_steps: int = 1, *,
                              lead_solver: str = "lu") -> TimeKKTPreconditioner:
    """Reference preconditioners.py:315-333 (lead_solver as in
    preconditioners.build_sweep: "lu" = the reference's SuperLU, "fastdiag" =
    the depth-free Kronecker-sum solve)."""
    st = sys.steady
    n_tau = st.n_terms if n_tau is None else n_tau
    z_op, sweep = build_sweep(st.triple.matrices[: st.n_terms], time_lead_terms(sys), partition, n_tau,
                              lead_solver=lead_solver, mass=st.mass)
    if mass_solver.startswith("cheb"):
        ms = make_mass_solver(st.mass, mass_solver, st.pattern, st.mass_slice)
    else:
        ms = make_mass_solver(st.mass, mass_solver)
    return TimeKKTPreconditioner(system=sys, mass_solve=ms, z_operator=z_op, sweep=sweep,
                                 richardson_steps=richardson_steps)
