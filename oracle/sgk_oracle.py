"""NumPy/SciPy restatement of the reference hot path (test infrastructure).

Inputs are plain SciPy CSR matrices and NumPy arrays in the reference's
matricized layout (N_h, N_xi); functions follow the reference's loop
structure (per-term CSR x dense, then the sparse right multiplication), so
their cost equals the reference's single-threaded CPU path.

Reference files: /root/reference/pkg/src/sgkkt/{operators,preconditioners,
krylov,linalg}.py.
"""

from __future__ import annotations

import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "cg",
    "chebyshev_mass_solve",
    "coupled_sweep_apply",
    "fgmres",
    "hgs_apply",
    "kron_apply",
    "kron_apply_rows",
    "kron_apply_sliced",
    "minres",
    "richardson_hgs",
    "shifted_lead",
    "splu_ref",
    "steady_kkt_apply",
    "steady_precond_apply",
    "time_kkt_apply",
    "time_lead",
    "time_precond_apply",
    "time_weights",
]


def _xh(x, h):
    """x @ h through the sparse path: (h^T x^T)^T (operators.py:53-55)."""
    return np.asarray((h.T @ x.T).T)


def kron_apply(couplings, operators, x):
    """operators.py:88-96: out = sum_t A_t x H_t, one term at a time."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    for h, a in zip(couplings, operators):
        out += _xh(a @ x, h)
    return out


def kron_apply_sliced(couplings, operators, x, src, dst, n_trunc):
    """operators.py:99-126."""
    slo, shi = src
    dlo, dhi = dst
    out = np.zeros((x.shape[0], dhi - dlo))
    if slo == shi or dlo == dhi:
        return out
    for h, a in zip(couplings[:n_trunc], operators[:n_trunc]):
        hs = h[slo:shi, dlo:dhi]
        if hs.nnz:
            out += _xh(a @ x[:, slo:shi], hs)
    return out


def splu_ref(mat):
    """linalg.py:103-120 (the factorization call, without the probe)."""
    return spla.splu(sp.csc_matrix(mat), diag_pivot_thresh=1.0)


def _ranges(boundaries):
    lo = 0
    out = []
    for hi in boundaries:
        out.append((lo, hi))
        lo = hi
    return out


def hgs_apply(couplings, terms, boundaries, n_tau, lead_lu, r):
    """HierarchicalGaussSeidel.apply, preconditioners.py:132-165."""
    n_xi = r.shape[1]

    def cross(v, src, dst):
        slo, shi = src
        dlo, dhi = dst
        acc = np.zeros((v.shape[0], dhi - dlo))
        if slo == shi:
            return acc
        for t in range(1, n_tau):
            hs = couplings[t][slo:shi, dlo:dhi]
            if hs.nnz:
                acc += _xh(terms[t] @ v[:, slo:shi], hs)
        return acc

    ranges = _ranges(boundaries)
    v = np.zeros_like(r)
    for lo, hi in ranges:
        v[:, lo:hi] = lead_lu.solve(r[:, lo:hi] - cross(v, (0, lo), (lo, hi)))
    for lo, hi in reversed(ranges[:-1]):
        rhs = r[:, lo:hi] - cross(v, (0, lo), (lo, hi)) - cross(v, (hi, n_xi), (lo, hi))
        v[:, lo:hi] = lead_lu.solve(rhs)
    return v


def richardson_hgs(couplings, terms, boundaries, n_tau, lead_lu, b, n_steps=1):
    """preconditioners.py:172-184."""
    x = hgs_apply(couplings, terms, boundaries, n_tau, lead_lu, b)
    for _ in range(n_steps - 1):
        x = x + hgs_apply(couplings, terms, boundaries, n_tau, lead_lu, b - kron_apply(couplings, terms, x))
    return x


def shifted_lead(mass, stiffness, beta, gamma):
    """preconditioners.py:187-195."""
    shift = np.sqrt((1.0 + gamma) / beta)
    return [(stiffness[0] + shift * mass).tocsr()] + [a.tocsr() for a in stiffness[1:]]


_ALPHA = 1.25
_RHO = 0.8


def chebyshev_mass_solve(mass, b, its=5):
    """preconditioners.py:70-98 (code sequence of omegas, not the paper's)."""
    diag = mass.diagonal()
    b = np.asarray(b, dtype=np.float64)
    scale = 1.0 / (_ALPHA * diag)
    if b.ndim == 2:
        scale = scale[:, None]
    x_prev = np.zeros_like(b)
    x = np.zeros_like(b)
    omega = 1.0
    for k in range(its):
        if k == 1:
            omega = 1.0 / (1.0 - _RHO**2 / 2.0)
        elif k > 1:
            omega = 1.0 / (1.0 - omega * _RHO**2 / 4.0)
        x_new = omega * (scale * (b - mass @ x) + x - x_prev) + x_prev
        x_prev, x = x, x_new
    return x


def steady_kkt_apply(mass, stiffness, couplings, weight_diag, beta, y, u, lam):
    """operators.py:181-194."""
    n_t = len(stiffness)
    a_lam = kron_apply(couplings[:n_t], stiffness, lam)
    a_y = kron_apply(couplings[:n_t], stiffness, y)
    r_y = (mass @ y) * weight_diag[None, :] - a_lam
    r_u = beta * (mass @ u) + mass @ lam
    r_lam = -a_y + mass @ u
    return r_y, r_u, r_lam


def steady_precond_apply(mass, stiffness, couplings, weight_diag, beta, gamma, boundaries, n_tau,
                         lead_lu, r_y, r_u, r_lam, mass_its=5, richardson_steps=1):
    """SteadyKKTPreconditioner.apply with Chebyshev mass solves
    (preconditioners.py:227-255)."""
    terms = shifted_lead(mass, stiffness, beta, gamma)
    cp = couplings[: len(stiffness)]
    v_y = chebyshev_mass_solve(mass, r_y, mass_its) / weight_diag[None, :]
    v_u = chebyshev_mass_solve(mass, r_u, mass_its) / beta
    z1 = richardson_hgs(cp, terms, boundaries, n_tau, lead_lu, r_lam, richardson_steps)
    w = (mass @ z1) * weight_diag[None, :]
    v_lam = richardson_hgs(cp, terms, boundaries, n_tau, lead_lu, w, richardson_steps)
    return v_y, v_u, v_lam


def coupled_sweep_apply(mass, stiffness, couplings, objective_weight, beta, boundaries, n_tau, kkt_lu,
                        r_y, r_u, r_lam):
    """CoupledSweepPreconditioner.apply, preconditioners.py:359-434."""
    n_h, n_xi = r_y.shape
    ident = couplings[0]

    def stiff(v, src, dst):
        slo, shi = src
        dlo, dhi = dst
        acc = np.zeros((n_h, dhi - dlo))
        if slo == shi:
            return acc
        for t in range(n_tau):
            hs = couplings[t][slo:shi, dlo:dhi]
            if hs.nnz:
                acc += _xh(stiffness[t] @ v[:, slo:shi], hs)
        return acc

    def massc(v, src, dst, h):
        slo, shi = src
        dlo, dhi = dst
        acc = np.zeros((n_h, dhi - dlo))
        if slo == shi:
            return acc
        hs = h[slo:shi, dlo:dhi]
        if hs.nnz:
            acc += _xh(mass @ v[:, slo:shi], hs)
        return acc

    vy = np.zeros((n_h, n_xi))
    vu = np.zeros((n_h, n_xi))
    vl = np.zeros((n_h, n_xi))

    def level(srcs, dst):
        dlo, dhi = dst
        ry = r_y[:, dlo:dhi].copy()
        ru = r_u[:, dlo:dhi].copy()
        rl = r_lam[:, dlo:dhi].copy()
        for src in srcs:
            ry -= massc(vy, src, dst, objective_weight)
            ry += stiff(vl, src, dst)
            ru -= beta * massc(vu, src, dst, ident)
            ru -= massc(vl, src, dst, ident)
            rl += stiff(vy, src, dst)
            rl -= massc(vu, src, dst, ident)
        sol = kkt_lu.solve(np.vstack([ry, ru, rl]))
        vy[:, dlo:dhi] = sol[:n_h]
        vu[:, dlo:dhi] = sol[n_h : 2 * n_h]
        vl[:, dlo:dhi] = sol[2 * n_h :]

    ranges = _ranges(boundaries)
    for lo, hi in ranges:
        level([(0, lo)], (lo, hi))
    for lo, hi in reversed(ranges[:-1]):
        level([(0, lo), (hi, n_xi)], (lo, hi))
    return vy, vu, vl


def fgmres(apply_op, apply_prec, b, tol, max_iters=500):
    """krylov.py:45-137 (right-preconditioned FGMRES, MGS + one conditional
    re-orthogonalisation, Givens, stop on |g_{j+1}|/||b||).
    Returns (x, iterations, converged, history)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    bn = np.linalg.norm(b)
    if bn == 0.0:
        raise ValueError("right-hand side must be nonzero")
    prec = apply_prec if apply_prec is not None else (lambda v: v)
    m_max = min(max_iters, n)
    V = np.empty((m_max + 1, n))
    Z = np.empty((m_max, n))
    H = np.zeros((m_max + 1, m_max))
    cs = np.zeros(m_max)
    sn = np.zeros(m_max)
    g = np.zeros(m_max + 1)
    g[0] = bn
    V[0] = b / bn
    hist = []
    conv = False
    its = 0
    for j in range(m_max):
        its = j + 1
        Z[j] = prec(V[j])
        w = np.array(apply_op(Z[j]), dtype=np.float64)
        w_in = np.linalg.norm(w)
        for i in range(j + 1):
            H[i, j] = V[i] @ w
            w -= H[i, j] * V[i]
        wn = np.linalg.norm(w)
        defect = np.abs(V[: j + 1] @ w).max() if wn > 0 else 0.0
        if wn == 0.0 or defect > 1e-8 * wn:
            for i in range(j + 1):
                c = V[i] @ w
                H[i, j] += c
                w -= c * V[i]
            wn = np.linalg.norm(w)
        H[j + 1, j] = wn
        brk = wn <= 1e-14 * max(w_in, 1e-300)
        if not brk:
            V[j + 1] = w / wn
        for i in range(j):
            a, bb = H[i, j], H[i + 1, j]
            H[i, j] = cs[i] * a + sn[i] * bb
            H[i + 1, j] = -sn[i] * a + cs[i] * bb
        d = np.hypot(H[j, j], H[j + 1, j])
        if d == 0.0:
            cs[j], sn[j] = 1.0, 0.0
        else:
            cs[j], sn[j] = H[j, j] / d, H[j + 1, j] / d
        H[j, j] = d
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        rr = abs(g[j + 1]) / bn
        hist.append(rr)
        if rr <= tol or brk:
            conv = True
            break
    y = np.zeros(its)
    for i in range(its - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1 : its] @ y[i + 1 : its]) / H[i, i]
    return Z[:its].T @ y, its, conv, np.array(hist)


def cg(apply_op, apply_prec, b, tol, max_iters=500):
    """Preconditioned CG from 0 with the 2-norm recurrence-residual test
    (new: the reference has no CG; pinned against scipy.sparse.linalg.cg)."""
    b = np.asarray(b, dtype=np.float64)
    bn = np.linalg.norm(b)
    if bn == 0.0:
        raise ValueError("right-hand side must be nonzero")
    prec = apply_prec if apply_prec is not None else (lambda v: v)
    x = np.zeros_like(b)
    r = b.copy()
    z = prec(r)
    p = z.copy()
    rz = r @ z
    hist = []
    conv = False
    it = 0
    for it in range(1, max_iters + 1):
        q = apply_op(p)
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        rel = np.linalg.norm(r) / bn
        hist.append(rel)
        if rel <= tol:
            conv = True
            break
        z = prec(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, it, conv, np.array(hist)


def minres(apply_op, apply_prec, b, tol, max_iters=500):
    """Preconditioned MINRES (Elman-Silvester-Wathen recurrence) with the
    true-2-norm residual tracked through A w (new: no reference)."""
    b = np.asarray(b, dtype=np.float64)
    bn = np.linalg.norm(b)
    if bn == 0.0:
        raise ValueError("right-hand side must be nonzero")
    prec = apply_prec if apply_prec is not None else (lambda v: v)
    n = b.size
    x = np.zeros(n)
    r = b.copy()
    v_old = np.zeros(n)
    v = b.copy()
    z = prec(v)
    gamma = np.sqrt(z @ v)
    gamma_old = 1.0
    eta = gamma
    s_old = s = 0.0
    c_old = c = 1.0
    w_old = np.zeros(n)
    w = np.zeros(n)
    aw_old = np.zeros(n)
    aw = np.zeros(n)
    hist = []
    conv = False
    it = 0
    for it in range(1, max_iters + 1):
        z = z / gamma
        az = apply_op(z)
        delta = az @ z
        v_new = az - (delta / gamma) * v - (gamma / gamma_old) * v_old
        z_new = prec(v_new)
        gamma_new = np.sqrt(z_new @ v_new)
        a0 = c * delta - c_old * s * gamma
        a1 = np.sqrt(a0 * a0 + gamma_new * gamma_new)
        a2 = s * delta + c_old * c * gamma
        a3 = s_old * gamma
        c_new, s_new = a0 / a1, gamma_new / a1
        w_new = (z - a3 * w_old - a2 * w) / a1
        aw_new = (az - a3 * aw_old - a2 * aw) / a1
        x = x + c_new * eta * w_new
        r = r - c_new * eta * aw_new
        eta = -s_new * eta
        rel = np.linalg.norm(r) / bn
        hist.append(rel)
        v_old, v, z = v, v_new, z_new
        w_old, w, aw_old, aw = w, w_new, aw, aw_new
        gamma_old, gamma = gamma, gamma_new
        c_old, c, s_old, s = c, c_new, s, s_new
        if rel <= tol:
            conv = True
            break
        if gamma == 0.0:
            break
    return x, it, conv, np.array(hist)


def timed(fn, *args, **kw):
    t0 = time.perf_counter()
    out = fn(*args, **kw)
    return out, time.perf_counter() - t0


def kron_apply_rows(couplings, operators, x, rows):
    """kron_apply restricted to a contiguous row slab [r0, r1) of the output
    (same per-term algorithm, operators.py:94-95); used for bounded CPU
    baseline samples."""
    r0, r1 = rows
    out = np.zeros((r1 - r0, x.shape[1]))
    for h, a in zip(couplings, operators):
        out += _xh(a[r0:r1] @ x, h)
    return out


# ---------------------------------------------------------------------------
# Time-dependent all-at-once KKT and the parallel-in-time preconditioner
# (reference operators.py:204-324, preconditioners.py:198-208, 278-333).
# Packed layout as in the reference: [y steps; u steps; lambda steps], each
# step an F-order (column-major) vec of an (N, n_xi) block.

def _split_time(v, n_t, n_h, n_xi):
    size = n_h * n_xi
    v = np.asarray(v, dtype=np.float64)
    return [np.stack([v[(b * n_t + k) * size:(b * n_t + k + 1) * size].reshape((n_h, n_xi), order="F")
                      for k in range(n_t)]) for b in range(3)]


def _join_time(y, u, lam):
    return np.concatenate([blk[k].reshape(-1, order="F") for blk in (y, u, lam) for k in range(blk.shape[0])])


def time_weights(n_t):
    """Trapezoid weights (1/2, 1, ..., 1, 1/2) and tau = 1/n_t (operators.py:212-223)."""
    w = np.ones(n_t)
    w[0] = 0.5
    w[-1] = 0.5
    return 1.0 / n_t, w


def time_kkt_apply(mass, stiffness, couplings, weight_diag, beta, n_t, v):
    """time_kkt_apply, operators.py:284-309."""
    n_h, n_xi = mass.shape[0], len(weight_diag)
    tau, w = time_weights(n_t)
    y, u, lam = _split_time(v, n_t, n_h, n_xi)
    cp = couplings[: len(stiffness)]
    step = lambda x: mass @ x + tau * kron_apply(cp, stiffness, x)
    ry, ru, rl = np.empty_like(y), np.empty_like(u), np.empty_like(lam)
    wd = weight_diag[None, :]
    for k in range(n_t):
        at_lam = step(lam[k])
        if k + 1 < n_t:
            at_lam -= mass @ lam[k + 1]
        ry[k] = tau * w[k] * ((mass @ y[k]) * wd) - at_lam
        ru[k] = beta * tau * w[k] * (mass @ u[k]) + tau * (mass @ lam[k])
        a_y = step(y[k])
        if k > 0:
            a_y -= mass @ y[k - 1]
        rl[k] = -a_y + tau * (mass @ u[k])
    return _join_time(ry, ru, rl)


def time_lead(mass, stiffness, beta, gamma, n_t):
    """time_lead_terms, preconditioners.py:198-208."""
    tau = 1.0 / n_t
    shift = 1.0 + tau * np.sqrt((1.0 + gamma) / beta)
    return [(shift * mass + tau * stiffness[0]).tocsr()] + [(tau * a).tocsr() for a in stiffness[1:]]


def time_precond_apply(mass, stiffness, couplings, weight_diag, beta, gamma, boundaries, n_tau, lead_lu, n_t, r,
                       mass_its=5, richardson_steps=1):
    """TimeKKTPreconditioner.apply, preconditioners.py:294-312 (Chebyshev mass solves)."""
    n_h, n_xi = mass.shape[0], len(weight_diag)
    tau, w = time_weights(n_t)
    terms = time_lead(mass, stiffness, beta, gamma, n_t)
    cp = couplings[: len(stiffness)]
    ry, ru, rl = _split_time(r, n_t, n_h, n_xi)
    wc = weight_diag[None, :]
    vy, vu, vl = np.empty_like(ry), np.empty_like(ru), np.empty_like(rl)
    for k in range(n_t):
        dk = w[k]
        vy[k] = chebyshev_mass_solve(mass, ry[k], mass_its) / (tau * dk * wc)
        vu[k] = chebyshev_mass_solve(mass, ru[k], mass_its) / (beta * tau * dk)
        z1 = richardson_hgs(cp, terms, boundaries, n_tau, lead_lu, rl[k], richardson_steps)
        ww = dk * (mass @ z1) * wc
        vl[k] = tau * richardson_hgs(cp, terms, boundaries, n_tau, lead_lu, ww, richardson_steps)
    return _join_time(vy, vu, vl)
