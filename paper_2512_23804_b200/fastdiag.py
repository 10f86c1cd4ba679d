"""Depth-free lead solves by fast diagonalisation.

The reference factors every lead block with SuperLU (linalg.py:103-120) and
the GPU path replays those factors as level-scheduled triangular solves
(linalg.py here, csrc/trisolve.cu): exact, but bounded by the factor's
dependency depth (config 5's P~: ~4.3k row levels).  For the BASELINE
problems the lead is a constant-coefficient Q1 operator on a uniform tensor
grid, i.e. a Kronecker sum

    A = K1 (x) M1 + M1 (x) K1   (shifted leads A_1 + c M included),
    M = M1 (x) M1,               node p = iy * n + ix,

so with the 1-D generalised eigenpairs K1 S = M1 S diag(mu), S^T M1 S = I the
lead, the shifted lead and the hGSoc block P~ (preconditioners.py:437-448)
are diagonal (3x3 block-diagonal) in the basis T = S (x) S.  A solve is then
four dense fp64 passes (cuBLAS DGEMMs) around one modal kernel
(csrc/fastdiag.cu) — no dependency chain at all.

The factor objects here are drop-ins for `LUFactors` in the `lead_factor` /
`kkt_factor` slots (reference seam: any object with ``.solve(b)``,
preconditioners.py:126,357): ``solve(b)`` on the host API and
``device_factors.solve_segments`` on the device path.  Results equal the LU
solves up to rounding (a different but backward-stable algorithm: see
tests/test_gpu_fastdiag.py for the measured agreement); the LU path stays the
default so parity with the reference is bit-for-bit in structure.

`kron_sum_split` refuses (ValueError) any matrix that is not such a Kronecker
sum to 1e-12 relative, so a variable-coefficient lead can never take this
path silently.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import torch
from scipy.sparse import csr_matrix

from . import _lib
from .device import _f64, as_device_state

__all__ = [
    "FastDiagFactors",
    "KRON_TOL",
    "fastdiag_factor",
    "fastdiag_kkt_factor",
    "is_kron_sum",
    "kron_sum_split",
]

KRON_TOL = 1e-12
# SGKKT_FD_HALF=0 keeps the full-size passes for centrosymmetric leads (A/B)
HALF = __import__("os").environ.get("SGKKT_FD_HALF", "1") != "0"


def _grid_side(n_rows: int) -> int:
    n = int(round(np.sqrt(n_rows)))
    if n * n != n_rows or n < 2:
        raise ValueError(f"{n_rows} unknowns are not an n x n tensor grid")
    return n


def _block(mat: csr_matrix, n: int, bi: int, bj: int) -> np.ndarray:
    return mat[bi * n:(bi + 1) * n, bj * n:(bj + 1) * n].toarray()


def kron_sum_split(a: sp.spmatrix, mass: sp.spmatrix) -> tuple[np.ndarray, np.ndarray]:
    """(K1, M1) with mass = M1 (x) M1 and a = K1 (x) M1 + M1 (x) K1 (node
    p = iy*n + ix), read off the leading n x n blocks and verified on every
    entry to KRON_TOL relative (max-norm).  ValueError otherwise."""
    a = sp.csr_matrix(a, dtype=np.float64)
    mass = sp.csr_matrix(mass, dtype=np.float64)
    if a.shape != mass.shape or a.shape[0] != a.shape[1]:
        raise ValueError("lead and mass matrices must be square and of one size")
    n = _grid_side(a.shape[0])
    m00 = float(mass[0, 0])
    if not m00 > 0.0:
        raise ValueError("mass matrix has a non-positive leading entry")
    m1 = _block(mass, n, 0, 0) / np.sqrt(m00)
    k00 = float(a[0, 0]) / (2.0 * m1[0, 0])
    k1 = (_block(a, n, 0, 0) - k00 * m1) / m1[0, 0]
    m1s, k1s = sp.csr_matrix(m1), sp.csr_matrix(k1)
    err_m = abs(sp.kron(m1s, m1s, format="csr") - mass).max()
    err_a = abs((sp.kron(k1s, m1s, format="csr") + sp.kron(m1s, k1s, format="csr")) - a).max()
    scale_m = abs(mass).max()
    scale_a = abs(a).max()
    if err_m > KRON_TOL * scale_m:
        raise ValueError(f"mass matrix is not M1 (x) M1 (rel. deviation {err_m / scale_m:.2e})")
    if err_a > KRON_TOL * scale_a:
        raise ValueError(f"lead is not a Kronecker sum K1 (x) M1 + M1 (x) K1 (rel. deviation {err_a / scale_a:.2e})")
    return 0.5 * (k1 + k1.T), 0.5 * (m1 + m1.T)


def is_kron_sum(a, mass) -> bool:
    try:
        kron_sum_split(a, mass)
    except ValueError:
        return False
    return True


@dataclass(frozen=True, eq=False)
class FastDiagFactors:
    """Modal factor of a Kronecker-sum lead (n_seg = 1) or of the hGSoc block
    P~ = [M 0 -A; 0 beta M M; -A M 0] (n_seg = 3).  Drop-in for LUFactors."""

    shape: tuple[int, int]
    n: int
    n_seg: int
    beta: float
    s: np.ndarray  # S (n x n), K1 S = M1 S diag(mu), S^T M1 S = I
    lam: np.ndarray  # mu_a + mu_b, a-major (n*n)
    ne: int = -1  # symmetric modes first (centrosymmetric butterfly form), -1: full passes
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    # the factor is its own device object (same seam as TriangularFactors)
    @property
    def device_factors(self) -> "FastDiagFactors":
        return self

    def _dev(self):
        d = self._cache.get("dev")
        if d is None:
            n_pad = -(-self.n // 8) * 8
            if n_pad > 256:
                raise ValueError("fastdiag: grid side above 255 is not supported by the device kernels")
            s_pad = np.zeros((n_pad, n_pad))
            s_pad[: self.n, : self.n] = self.s
            s_t = _f64(s_pad)
            lam_t = _f64(self.lam)
            keep = [s_t, lam_t]
            ne, hp, sh = 0, 0, None
            h = self.n // 2
            if self.ne >= 0 and HALF and -(-(h + 1) // 8) * 8 <= 128:
                ne = self.ne
                hp = -(-(h + 1) // 8) * 8
                halves = np.zeros((2, hp, hp))
                halves[0, : h + self.n % 2, :ne] = self.s[: h + self.n % 2, :ne]
                halves[1, :h, : self.n - ne] = self.s[:h, ne:]
                sh_t = _f64(halves)
                keep.append(sh_t)
                sh = sh_t.data_ptr()
            st = _lib.FastDiag(n=self.n, n_seg=self.n_seg, np=n_pad, pad=0, s=s_t.data_ptr(),
                               lam=lam_t.data_ptr(), beta=float(self.beta), ne=ne, hp=hp, sh=sh)
            d = (st, keep)
            self._cache["dev"] = d
        return d[0]

    def solve_segments(self, b_segs, x_segs, width: int, stream=None) -> None:
        """x = A^-1 b (or P~^-1 on the (y, u, lambda) segments) on `width`
        columns; same contract as TriangularFactors.solve_segments."""
        if width == 0:
            return
        if len(b_segs) != self.n_seg or len(x_segs) != self.n_seg:
            raise ValueError(f"factor takes {self.n_seg} row segment(s)")
        seg_rows = self.n * self.n

        def segview(segs):
            ptrs = (ctypes.c_void_p * 3)()
            ld = col0 = None
            for i, (t, c0) in enumerate(segs):
                if t.shape[0] != seg_rows or t.dtype != torch.float64 or not t.is_cuda or t.stride(1) != 1:
                    raise ValueError("segment must be a (n*n, cols) float64 CUDA tensor")
                if c0 + width > t.shape[1]:
                    raise ValueError("segment too narrow")
                if ld is None:
                    ld, col0 = t.stride(0), c0
                elif ld != t.stride(0) or col0 != c0:
                    raise ValueError("segments must share leading dimension and column offset")
                ptrs[i] = t.data_ptr()
            return _lib.SegView(ptr=ptrs, ld=ld, col0=col0, seg_rows=seg_rows)

        bv, xv = segview(b_segs), segview(x_segs)
        st = self._dev()
        lib = _lib.lib()
        n_work = int(lib.sgk_fastdiag_work_doubles(ctypes.byref(st), int(width)))
        sp_ = _lib.stream_ptr(stream)
        # scratch reused per stream (stream order serialises its users; grown
        # on demand) instead of an allocation per solve
        key = ("work", sp_)
        work = self._cache.get(key)
        if work is None or work.numel() < n_work or work.device != b_segs[0][0].device:
            work = torch.empty(max(n_work, 1), dtype=torch.float64, device=b_segs[0][0].device)
            if stream is not None:
                work.record_stream(stream)
            self._cache[key] = work
        rc = lib.sgk_fastdiag_solve(ctypes.byref(st), ctypes.byref(bv), ctypes.byref(xv), work.data_ptr(),
                                    int(width), sp_)
        _lib.check(rc, "sgk_fastdiag_solve")

    def solve(self, b):
        """A^-1 b for b of shape (n,) or (n, k) (LUFactors.solve contract,
        reference linalg.py:83-87); NumPy in -> NumPy out."""
        if tuple(b.shape)[0] != self.shape[0]:
            raise ValueError("right-hand side length does not match factor size")
        vec = len(b.shape) == 1
        bd, host = as_device_state(b)
        b2 = bd.reshape(self.shape[0], -1).contiguous()
        x = torch.empty_like(b2)
        rows = self.n * self.n
        segs_b = [(b2[i * rows:(i + 1) * rows], 0) for i in range(self.n_seg)]
        segs_x = [(x[i * rows:(i + 1) * rows], 0) for i in range(self.n_seg)]
        self.solve_segments(segs_b, segs_x, b2.shape[1])
        out = x.reshape(-1) if vec else x
        if host:
            return out.to("cpu") if isinstance(b, torch.Tensor) else out.cpu().numpy()
        return out


CENTRO_TOL = 1e-10  # eigh leaves ~1e-12 asymmetry in the A_1 modes (n = 127)


def _centro_order(s: np.ndarray):
    """Mode order for the centrosymmetric (butterfly) kernels: when every
    1-D mode is symmetric or antisymmetric (S[n-1-i, j] = +-S[i, j] to
    CENTRO_TOL relative — true for the symmetric Toeplitz K1, M1 of a
    uniform grid), the permutation putting the symmetric modes first and
    their count; else None (full passes)."""
    n = s.shape[0]
    flip = s[::-1, :]
    norm = np.linalg.norm(s, axis=0)
    par = np.sign(np.einsum("ij,ij->j", flip, s))
    if np.any(par == 0) or np.max(np.linalg.norm(flip - par[None, :] * s, axis=0) / norm) > CENTRO_TOL:
        return None
    perm = np.concatenate([np.nonzero(par > 0)[0], np.nonzero(par < 0)[0]])
    return perm, int(np.sum(par > 0))


def _modal(a, mass):
    k1, m1 = kron_sum_split(a, mass)
    mu, s = scipy.linalg.eigh(k1, m1)
    n = len(mu)
    ne = -1
    co = _centro_order(s)
    if co is not None:
        perm, ne = co
        s, mu = s[:, perm], mu[perm]
    lam = (mu[:, None] + mu[None, :]).reshape(-1)
    return n, np.ascontiguousarray(s), np.ascontiguousarray(lam), ne


def fastdiag_factor(a: sp.spmatrix, mass: sp.spmatrix) -> FastDiagFactors:
    """Factor of a Kronecker-sum lead (A_1, or A_1 + c M): drop-in for
    sparse_lu(a) in the hGS lead slot (preconditioners.py:211-224)."""
    n, s, lam, ne = _modal(a, mass)
    if np.any(lam <= 0.0):
        raise ValueError("lead is not positive definite")
    return FastDiagFactors(shape=a.shape, n=n, n_seg=1, beta=0.0, s=s, lam=lam, ne=ne)


def fastdiag_kkt_factor(a1: sp.spmatrix, mass: sp.spmatrix, beta: float) -> FastDiagFactors:
    """Factor of P~ = [M 0 -A_1; 0 beta M M; -A_1 M 0]: drop-in for
    sparse_lu(deterministic_kkt_matrix(sys)) (preconditioners.py:451-462)."""
    if not beta > 0.0:
        raise ValueError("beta must be positive")
    n, s, lam, ne = _modal(a1, mass)
    rows = 3 * n * n
    return FastDiagFactors(shape=(rows, rows), n=n, n_seg=3, beta=float(beta), s=s, lam=lam, ne=ne)
