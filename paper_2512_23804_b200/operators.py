"""Galerkin operators on the B200: drop-in for `sgkkt.operators`
(reference pkg/src/sgkkt/operators.py).

States are (N_h, N_xi) float64 matrices in the reference's matricized sense
(column k = chaos mode psi_k).  On the device they are stored node-major
(row-major (N_h, N_xi): the chaos coefficients of one mesh node are
contiguous), which is what the fused kernel streams.  Every function accepts

* a CUDA tensor  -> computes on the device, returns a CUDA tensor;
* a NumPy array  -> copies it to the device, computes, returns NumPy (the
  reference-facing path; host<->device copies included);
* a pinned CPU tensor -> as NumPy but with asynchronous DMA, returns a CPU
  tensor (or writes into ``out``).

There is no CPU fallback: without libsgkkt_b200.so or a CUDA device every
call raises RuntimeError.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch
from scipy.sparse import csr_matrix

from .basis import TripleProductSet
from .device import DevicePattern, DeviceProgram, as_device_state, device, run_program
from . import device as _dev
from .program import Coupling, compile_program, coupling_from_csr

__all__ = [
    "KroneckerSumOperator",
    "SteadyKKT",
    "kron_apply",
    "kron_apply_sliced",
    "matricize",
    "right_multiply",
    "steady_kkt_apply",
    "steady_rhs",
    "to_host",
    "vectorize",
]


def matricize(v, n_h: int, n_xi: int):
    """Column-major reshape of a packed vector (reference operators.py:41-46)."""
    if isinstance(v, torch.Tensor):
        if v.numel() != n_h * n_xi:
            raise ValueError(f"expected length {n_h * n_xi}, got {v.numel()}")
        return v.reshape(n_xi, n_h).T
    v = np.asarray(v, dtype=np.float64)
    if v.size != n_h * n_xi:
        raise ValueError(f"expected length {n_h * n_xi}, got {v.size}")
    return v.reshape((n_h, n_xi), order="F")


def vectorize(x):
    """Inverse of matricize (reference operators.py:49-50)."""
    if isinstance(x, torch.Tensor):
        return x.T.reshape(-1)
    return np.asarray(x).reshape(-1, order="F")


def right_multiply(x, h: csr_matrix):
    """x @ h for a host state (reference operators.py:53-55); host helper."""
    return np.asarray((h.T @ np.asarray(x).T).T)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").numpy()


def _finish(out: torch.Tensor, host: bool, like, out_arg=None):
    """Return in the caller's flavour (device tensor, NumPy or CPU tensor)."""
    if out_arg is not None:
        if isinstance(out_arg, torch.Tensor):
            out_arg.copy_(out, non_blocking=out_arg.is_pinned())
            if not out_arg.is_cuda:
                torch.cuda.current_stream().synchronize()
            return out_arg
        np.copyto(out_arg, to_host(out))
        return out_arg
    if not host:
        return out
    if isinstance(like, torch.Tensor):
        return out.to("cpu")
    return to_host(out)


@dataclass(frozen=True, eq=False)
class KroneckerSumOperator:
    """sum_l couplings[l] (x) operators[l] (reference operators.py:58-85).

    The device side stores the operators on ONE CSR pattern with t-stacked
    values and compiles the coupling matrices into programs on first use."""

    couplings: list[csr_matrix]
    operators: list[csr_matrix]
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if len(self.couplings) != len(self.operators):
            raise ValueError("term counts differ")
        if not self.couplings:
            raise ValueError("need at least one term")
        n_xi = self.couplings[0].shape[0]
        n_h = self.operators[0].shape[0]
        for h in self.couplings:
            if h.shape != (n_xi, n_xi):
                raise ValueError("coupling matrices must share their size")
        for a in self.operators:
            if a.shape != (n_h, n_h):
                raise ValueError("operator matrices must share their size")

    @property
    def n_terms(self) -> int:
        return len(self.couplings)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.operators[0].shape[0], self.couplings[0].shape[0])

    # -- device state ------------------------------------------------------
    @property
    def pattern(self) -> DevicePattern:
        pat = self._cache.get("pattern")
        if pat is None:
            from .gpu_setup import attached_pattern

            pat = attached_pattern(self.operators) or DevicePattern(list(self.operators))
            self._cache["pattern"] = pat
        return pat

    def program(self, src_ranges, dst, t_lo: int, t_hi: int, scale: float = 1.0) -> DeviceProgram:
        """Program for out[:, dst] = scale * sum_{t in [t_lo,t_hi)} A_t V[:, src] H_t[src, dst]."""
        key = ("prog", tuple(src_ranges), tuple(dst), t_lo, t_hi, scale)
        prog = self._cache.get(key)
        if prog is None:
            cps = []
            for t in range(t_lo, t_hi):
                h = self.couplings[t].tocsr()
                for src in src_ranges:
                    cps.append(coupling_from_csr(0, 0, t, h, src, dst, scale))
            prog = DeviceProgram(cps, (dst[1] - dst[0],), n_inputs=1)
            self._cache[key] = prog
        return prog

    def algorithmic_bytes(self) -> int:
        """Bytes one full matvec must move at least once:
        V read + W written + t-stacked values + int32 pattern + H_t."""
        n_h, n_xi = self.shape
        nnz_h = sum(int(h.nnz) for h in self.couplings)
        pat = self.pattern
        return 16 * n_h * n_xi + pat.algorithmic_bytes + 12 * nnz_h


def _slab_plan(op: KroneckerSumOperator, n_slabs: int):
    """Row slabs [a, b) and, per slab, the last input row its stencil reads."""
    key = ("slabs", n_slabs)
    plan = op._cache.get(key)
    if plan is None:
        pat = op.pattern
        n = pat.n_rows
        edges = np.linspace(0, n, n_slabs + 1).astype(np.int64)
        need = []
        for a, b in zip(edges[:-1], edges[1:]):
            cols = pat.indices[pat.indptr[a]:pat.indptr[b]]
            need.append(int(cols.max()) + 1 if cols.size else int(b))
        plan = (edges, need)
        op._cache[key] = plan
    return plan


def _kron_apply_pipelined(op: KroneckerSumOperator, x_cpu: torch.Tensor, out_cpu: torch.Tensor,
                          n_slabs: int = 32) -> torch.Tensor:
    """Host buffers in and out (pinned): H2D of row slab s+1, the matvec of
    slab s and the D2H of slab s-1 run on three streams at once, so the two
    PCIe directions and the kernel overlap (the end-to-end path)."""
    n_h, n_xi = op.shape
    dev = device()
    st = op._cache.get("streams")
    if st is None:
        st = tuple(torch.cuda.Stream(device=dev) for _ in range(3))
        op._cache["streams"] = st
    s_in, s_cmp, s_out = st
    # staging buffers per call from the caching allocator (allocated on the
    # current stream, which every pipeline stream waits on below; the current
    # stream waits for the last D2H before they are released)
    xd = torch.empty((n_h, n_xi), dtype=torch.float64, device=dev)
    wd = torch.empty((n_h, n_xi), dtype=torch.float64, device=dev)
    n_slabs = max(1, min(int(n_slabs), n_h))
    edges, need = _slab_plan(op, n_slabs)
    prog = op.program([(0, n_xi)], (0, n_xi), 0, op.n_terms)
    cur = torch.cuda.current_stream(dev)
    for s_ in st:
        s_.wait_stream(cur)
    ev_in = []
    for a, b in zip(edges[:-1], edges[1:]):
        with torch.cuda.stream(s_in):
            xd[a:b].copy_(x_cpu[a:b], non_blocking=True)
            e = torch.cuda.Event()
            e.record(s_in)
            ev_in.append(e)
    done = 0
    for k, (a, b) in enumerate(zip(edges[:-1], edges[1:])):
        while done < len(ev_in) and edges[done] < need[k]:
            s_cmp.wait_event(ev_in[done])
            done += 1
        run_program(op.pattern, prog, [(xd, 0)], [(wd, 0)], alpha=[1.0], beta=[0.0], stream=s_cmp,
                    rows=(int(a), int(b)))
        e = torch.cuda.Event()
        e.record(s_cmp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(e)
            out_cpu[a:b].copy_(wd[a:b], non_blocking=True)
    cur.wait_stream(s_out)
    s_out.synchronize()
    return out_cpu


def _pipeline_ok(op: KroneckerSumOperator) -> bool:
    """The slab pipeline needs row-range launches, i.e. the full-column
    program must compile to the 9-point fast path (a many-term operator such
    as config 3 does not: it takes the plain device path)."""
    ok = op._cache.get("pipeline_ok")
    if ok is None:
        n_xi = op.shape[1]
        ok = bool(_dev.FAST9 and op.pattern.pattern9() is not None
                  and op.program([(0, n_xi)], (0, n_xi), 0, op.n_terms).fast9(op.pattern.n_slices) is not None)
        op._cache["pipeline_ok"] = ok
    return ok


def kron_apply(op: KroneckerSumOperator, x, out=None, n_slabs: int = 32):
    """W = sum_t A_t X H_t (reference operators.py:88-96), one fused launch.
    Pinned host tensors in/out (contiguous, float64) take the overlapped slab
    pipeline."""
    n_h, n_xi = op.shape
    if (isinstance(x, torch.Tensor) and not x.is_cuda and x.is_pinned() and isinstance(out, torch.Tensor)
            and not out.is_cuda and out.is_pinned() and out.is_contiguous()
            and tuple(x.shape) == (n_h, n_xi) and tuple(out.shape) == (n_h, n_xi) and x.dtype == torch.float64
            and out.dtype == torch.float64 and _pipeline_ok(op)):
        return _kron_apply_pipelined(op, x.contiguous(), out, n_slabs)
    xd, host = as_device_state(x, (n_h, n_xi))
    w = torch.empty((n_h, n_xi), dtype=torch.float64, device=xd.device)
    prog = op.program([(0, n_xi)], (0, n_xi), 0, op.n_terms)
    run_program(op.pattern, prog, [(xd, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
    return _finish(w, host, x, out)


def kron_apply_sliced(op: KroneckerSumOperator, x, src_cols, dst_cols, n_trunc: int):
    """sum_{t<n_trunc} A_t X[:, src] H_t[src, dst] (reference operators.py:99-126)."""
    slo, shi = src_cols
    dlo, dhi = dst_cols
    n_h, n_xi = op.shape
    if not (0 <= slo <= shi <= n_xi and 0 <= dlo <= dhi <= n_xi):
        raise ValueError("column ranges out of bounds")
    if not 1 <= n_trunc <= op.n_terms:
        raise ValueError("truncation count out of range")
    xd, host = as_device_state(x, (n_h, n_xi))
    out = torch.empty((n_h, dhi - dlo), dtype=torch.float64, device=xd.device)
    if dhi > dlo:
        prog = op.program([(slo, shi)], (dlo, dhi), 0, n_trunc)
        run_program(op.pattern, prog, [(xd, 0)], [(out, 0)], alpha=[1.0], beta=[0.0])
    return _finish(out, host, x)


@dataclass(frozen=True, eq=False)
class SteadyKKT:
    """Steady optimal-control KKT operator (reference operators.py:129-178).

        [ M (x) H^gamma    0            -A^T ] [Y]
        [ 0                beta M (x) I  M   ] [U]
        [ -A               M (x) I       0   ] [L]      A = sum_t H_t (x) A_t
    """

    mass: csr_matrix
    stiffness: list[csr_matrix]
    triple: TripleProductSet
    beta: float
    gamma: float
    target: np.ndarray
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if self.beta <= 0:
            raise ValueError("beta must be positive")
        if self.gamma < 0:
            raise ValueError("gamma must be nonnegative")
        if abs(self.gamma - self.triple.gamma) > 1e-14:
            raise ValueError("gamma disagrees with the triple-product weights")
        if len(self.stiffness) > self.triple.n_terms:
            raise ValueError("more stiffness terms than coupling matrices")
        if np.asarray(self.target).shape != (self.n_h, self.n_xi):
            raise ValueError("target shape does not match the system")

    @property
    def n_h(self) -> int:
        return self.mass.shape[0]

    @property
    def n_xi(self) -> int:
        return self.triple.size

    @property
    def n_terms(self) -> int:
        return len(self.stiffness)

    def stiffness_operator(self) -> KroneckerSumOperator:
        op = self._cache.get("a_op")
        if op is None:
            op = KroneckerSumOperator(couplings=self.triple.matrices[: self.n_terms], operators=self.stiffness)
            self._cache["a_op"] = op
        return op

    def block_size(self) -> int:
        return self.n_h * self.n_xi

    # -- device state ------------------------------------------------------
    @property
    def pattern(self) -> DevicePattern:
        """Slices [A_0 .. A_{T-1}, M] on one pattern (M is slice T)."""
        pat = self._cache.get("pattern")
        if pat is None:
            from .gpu_setup import attached_pattern

            mats = list(self.stiffness) + [self.mass]
            pat = attached_pattern(mats) or DevicePattern(mats)
            self._cache["pattern"] = pat
        return pat

    @property
    def mass_slice(self) -> int:
        return self.n_terms

    def kkt_program(self) -> DeviceProgram:
        prog = self._cache.get("kkt_prog")
        if prog is None:
            n_xi, T, m = self.n_xi, self.n_terms, self.mass_slice
            full = (0, n_xi)
            wdiag = self.triple.objective_weight.tocsr()
            eye = sp.identity(n_xi, format="csr")
            cps: list[Coupling | None] = []
            # inputs: 0=Y, 1=U, 2=L ; outputs: 0=r_y, 1=r_u, 2=r_l
            cps.append(coupling_from_csr(0, 0, m, wdiag, full, full, 1.0))  # (M Y) diag(h^gamma)
            for t in range(T):
                h = self.triple.matrices[t].tocsr()
                cps.append(coupling_from_csr(2, 0, t, h, full, full, -1.0))  # - A^T L (A symmetric use, ops.py:188)
                cps.append(coupling_from_csr(0, 2, t, h, full, full, -1.0))  # - A Y
            cps.append(coupling_from_csr(1, 1, m, eye, full, full, self.beta))  # beta M U
            cps.append(coupling_from_csr(2, 1, m, eye, full, full, 1.0))  # M L
            cps.append(coupling_from_csr(1, 2, m, eye, full, full, 1.0))  # M U
            prog = DeviceProgram(cps, (n_xi, n_xi, n_xi), n_inputs=3)
            self._cache["kkt_prog"] = prog
        return prog

    def kkt_programs_split(self) -> tuple[DeviceProgram, DeviceProgram]:
        """The KKT matvec as two launches: the stiffness-coupled inputs (Y, L:
        2 x ceil(n_xi/128) column groups <= 8 -> the warp-specialised 9-point
        kernel) writing all three outputs, then the mass-only input U
        accumulated into r_u and r_l (init = the outputs)."""
        progs = self._cache.get("kkt_split")
        if progs is None:
            n_xi, T, m = self.n_xi, self.n_terms, self.mass_slice
            full = (0, n_xi)
            wdiag = self.triple.objective_weight.tocsr()
            eye = sp.identity(n_xi, format="csr")
            cps: list[Coupling | None] = []
            # inputs: 0=Y, 1=L ; outputs: 0=r_y, 1=r_u, 2=r_l
            cps.append(coupling_from_csr(0, 0, m, wdiag, full, full, 1.0))  # (M Y) diag(h^gamma)
            for t in range(T):
                h = self.triple.matrices[t].tocsr()
                cps.append(coupling_from_csr(1, 0, t, h, full, full, -1.0))  # - A^T L
                cps.append(coupling_from_csr(0, 2, t, h, full, full, -1.0))  # - A Y
            cps.append(coupling_from_csr(1, 1, m, eye, full, full, 1.0))  # M L
            p_yl = DeviceProgram(cps, (n_xi, n_xi, n_xi), n_inputs=2)
            cps_u = [coupling_from_csr(0, 0, m, eye, full, full, self.beta),  # r_u += beta M U
                     coupling_from_csr(0, 1, m, eye, full, full, 1.0)]  # r_l += M U
            p_u = DeviceProgram(cps_u, (n_xi, n_xi), n_inputs=1)
            progs = (p_yl, p_u)
            self._cache["kkt_split"] = progs
        return progs

    def algorithmic_bytes(self) -> int:
        """KKT matvec floor: 3 blocks read + 3 written + (T+1) value slices."""
        nnz_h = sum(int(h.nnz) for h in self.triple.matrices[: self.n_terms])
        return 48 * self.n_h * self.n_xi + self.pattern.algorithmic_bytes + 12 * (nnz_h + 2 * self.n_xi)


# SGKKT_KKT_SPLIT=1: the KKT matvec as two launches (Y/L couplings on the
# warp-specialised kernel + a mass-only launch for U) instead of one 3-input
# launch (12 column groups at config 5 -> the alternating 16-warp kernel).
# Measured at config 5: 0.594 ms split vs 0.446 ms fused (tools/time_kkt.py),
# so the fused launch stays the default.
KKT_SPLIT = __import__("os").environ.get("SGKKT_KKT_SPLIT", "0") == "1"


def steady_kkt_apply_device(sys: SteadyKKT, y: torch.Tensor, u: torch.Tensor, lam: torch.Tensor,
                            out: tuple[torch.Tensor, torch.Tensor, torch.Tensor]) -> None:
    if KKT_SPLIT and sys.n_xi > 128:
        p_yl, p_u = sys.kkt_programs_split()
        run_program(sys.pattern, p_yl, [(y, 0), (lam, 0)], [(out[0], 0), (out[1], 0), (out[2], 0)],
                    alpha=[1.0] * 3, beta=[0.0] * 3)
        run_program(sys.pattern, p_u, [(u, 0)], [(out[1], 0), (out[2], 0)], [(out[1], 0), (out[2], 0)],
                    alpha=[1.0] * 2, beta=[1.0] * 2)
        return
    run_program(sys.pattern, sys.kkt_program(), [(y, 0), (u, 0), (lam, 0)],
                [(out[0], 0), (out[1], 0), (out[2], 0)], alpha=[1.0] * 3, beta=[0.0] * 3)


def steady_kkt_apply(sys: SteadyKKT, y, u, lam):
    """The three block rows of the KKT operator (reference operators.py:181-194),
    fused into one pass over the shared pattern."""
    shape = (sys.n_h, sys.n_xi)
    blocks = []
    host = False
    for name, blk in (("y", y), ("u", u), ("lam", lam)):
        if tuple(blk.shape) != shape:
            raise ValueError(f"block {name} has shape {tuple(blk.shape)}, expected {shape}")
        d, h = as_device_state(blk, shape)
        blocks.append(d)
        host = host or h
    outs = tuple(torch.empty(shape, dtype=torch.float64, device=blocks[0].device) for _ in range(3))
    steady_kkt_apply_device(sys, *blocks, outs)
    return tuple(_finish(o, host, y) for o in outs)


def steady_rhs(sys: SteadyKKT):
    """(M Y_d, 0, 0) (reference operators.py:197-201) — host setup."""
    b_y = np.asarray(sys.mass @ np.asarray(sys.target))
    zero = np.zeros((sys.n_h, sys.n_xi))
    return b_y, zero, zero.copy()
