"""The host half of the LU path: SuperLU factor extraction, permutation
conventions and level schedules, checked by a NumPy emulation of the device
algorithm (csrc/trisolve.cu) against SuperLU.solve (CPU only)."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from paper_2512_23804_b200.linalg import SingularMatrixError, csr_from_coo, level_schedule, sparse_lu
from paper_2512_23804_b200.problems import build_problem, steady_system


def emulate_trisolve(lu, b):
    """Row-by-row in level order exactly as the kernels do: factor row k
    reads b[in_perm[k]]; U rows write x[out_perm[k]]."""
    L = sp.tril(sp.csr_matrix(lu.L), k=-1, format="csr")
    U = sp.csr_matrix(lu.U)
    d = U.diagonal()
    U = sp.triu(U, k=1, format="csr")
    in_perm = np.argsort(lu.perm_r)
    out_perm = np.argsort(lu.perm_c)
    ol, _ = level_schedule(L, lower=True)
    ou, _ = level_schedule(U, lower=False)
    n = b.shape[0]
    z = np.zeros_like(b)
    done = np.zeros(n, bool)
    for k in ol:
        cols = L.indices[L.indptr[k]:L.indptr[k + 1]]
        assert done[cols].all()
        z[k] = b[in_perm[k]] - L.data[L.indptr[k]:L.indptr[k + 1]] @ z[cols]
        done[k] = True
    x = np.zeros_like(b)
    done[:] = False
    for k in ou:
        cols = U.indices[U.indptr[k]:U.indptr[k + 1]]
        assert done[cols].all()
        z[k] = (z[k] - U.data[U.indptr[k]:U.indptr[k + 1]] @ z[cols]) / d[k]
        x[out_perm[k]] = z[k]
        done[k] = True
    return x


@pytest.mark.parametrize("kind", ["random", "kkt"])
def test_superlu_convention_and_schedule(rng, kind):
    if kind == "random":
        a = sp.random(60, 60, density=0.1, random_state=3, format="csr") + 4 * sp.eye(60)
    else:
        b = build_problem(2, n=8)
        s = steady_system(b)
        a = sp.bmat([[s.mass, None, -s.stiffness[0]], [None, s.beta * s.mass, s.mass],
                     [-s.stiffness[0], s.mass, None]], format="csr")
    lu = spla.splu(sp.csc_matrix(a), diag_pivot_thresh=1.0)
    rhs = rng.standard_normal((a.shape[0], 3))
    want = lu.solve(rhs)
    got = emulate_trisolve(lu, rhs)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


def test_level_schedule_depth():
    lower = sp.csr_matrix(np.tril(np.ones((5, 5)), -1))
    order, depth = level_schedule(lower, lower=True)
    assert depth == 5 and list(order) == [0, 1, 2, 3, 4]
    diag_only = sp.csr_matrix((4, 4))
    assert level_schedule(diag_only, lower=True)[1] == 1


def test_singular_matrix_named():
    a = csr_from_coo(3, 3, [0, 1, 2], [0, 1, 1], [1.0, 2.0, 3.0])
    with pytest.raises(SingularMatrixError):
        sparse_lu(a)


def test_csr_from_coo_validation():
    with pytest.raises(ValueError):
        csr_from_coo(2, 2, [2], [0], [1.0])
    m = csr_from_coo(2, 2, [0, 0, 1], [1, 1, 0], [1.0, 2.0, 5.0])
    assert m[0, 1] == 3.0 and m.nnz == 2


def emulate_grouped(lu, b):
    """NumPy emulation of sgk_trisolve_grouped: group tasks in level order,
    outside contributions first, then the in-group chain."""
    from paper_2512_23804_b200.linalg import chain_groups, grouped_triangles

    L = sp.tril(sp.csr_matrix(lu.L), k=-1, format="csr")
    U = sp.csr_matrix(lu.U)
    d = U.diagonal()
    U = sp.triu(U, k=1, format="csr")
    for m in (L, U):
        m.sort_indices()
    (lt, lw, lio, _), (ut, uw, uio, udinv) = grouped_triangles(L, U, d, np.argsort(lu.perm_r), np.argsort(lu.perm_c))
    n = b.shape[0]
    work = np.zeros_like(b)
    x = np.zeros_like(b)
    for tri, wrow, iorow, dinv, fwd in ((lt, lw, lio, None, True), (ut, uw, uio, udinv, False)):
        gptr, order, _ = chain_groups(tri)
        done = np.zeros(n, bool)
        for g in order:
            r0, r1 = gptr[g], gptr[g + 1]
            part = {}
            for p in range(r0, r1):
                cols = tri.indices[tri.indptr[p]:tri.indptr[p + 1]]
                vals = tri.data[tri.indptr[p]:tri.indptr[p + 1]]
                out = cols < r0
                assert done[cols[out]].all()
                init = b[iorow[p]] if fwd else work[wrow[p]]
                part[p] = init - vals[out] @ work[wrow[cols[out]]]
            for p in range(r0, r1):
                cols = tri.indices[tri.indptr[p]:tri.indptr[p + 1]]
                vals = tri.data[tri.indptr[p]:tri.indptr[p + 1]]
                inn = cols >= r0
                y = part[p] - vals[inn] @ work[wrow[cols[inn]]]
                if not fwd:
                    y = y * dinv[p]
                    x[iorow[p]] = y
                work[wrow[p]] = y
                done[p] = True
    return x


@pytest.mark.parametrize("kind", ["random", "kkt"])
def test_grouped_trisolve_emulation(rng, kind):
    if kind == "random":
        a = sp.random(80, 80, density=0.08, random_state=5, format="csr") + 4 * sp.eye(80)
    else:
        b = build_problem(2, n=8)
        s = steady_system(b)
        a = sp.bmat([[s.mass, None, -s.stiffness[0]], [None, s.beta * s.mass, s.mass],
                     [-s.stiffness[0], s.mass, None]], format="csr")
    lu = spla.splu(sp.csc_matrix(a), diag_pivot_thresh=1.0)
    rhs = rng.standard_normal((a.shape[0], 2))
    want = lu.solve(rhs)
    got = emulate_grouped(lu, rhs)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


def emulate_group_blocks(strict, dinv, gptr, order, mptr, minv, rhs):
    """NumPy emulation of trsv_group on a processing-space lower triangle:
    groups in ticket order, outside contributions, then the dense in-group
    inverse block (csrc/trisolve.cu phases 1-2)."""
    n = strict.shape[0]
    y = np.full_like(rhs, np.nan)
    for g in order:
        a, b = int(gptr[g]), int(gptr[g + 1])
        part = rhs[a:b].copy()
        for r in range(a, b):
            lo, hi = strict.indptr[r], strict.indptr[r + 1]
            cols, vals = strict.indices[lo:hi], strict.data[lo:hi]
            out = cols < a
            assert not np.isnan(y[cols[out]]).any(), "dependency not finished"
            part[r - a] -= vals[out] @ y[cols[out]]
        m = b - a
        blk = minv[mptr[g]:mptr[g] + m * m].reshape(m, m)
        y[a:b] = blk @ part
    return y


@pytest.mark.parametrize("upper", [False, True])
def test_grouped_inverse_blocks_solve_the_triangle(rng, upper):
    from paper_2512_23804_b200.linalg import chain_groups, group_dependencies, group_inverses

    b = build_problem(2, n=8)
    s = steady_system(b)
    a = sp.bmat([[s.mass, None, -s.stiffness[0]], [None, s.beta * s.mass, s.mass],
                 [-s.stiffness[0], s.mass, None]], format="csr")
    lu = spla.splu(sp.csc_matrix(a), diag_pivot_thresh=1.0)
    if upper:  # U reversed into a lower triangle, as grouped_triangles does
        u = sp.csr_matrix(lu.U)
        n = u.shape[0]
        rev = np.arange(n)[::-1]
        t = sp.csr_matrix(u.toarray()[np.ix_(rev, rev)])
        dinv = 1.0 / t.diagonal()
        strict = sp.tril(t, k=-1, format="csr")
        full = t
    else:
        strict = sp.tril(sp.csr_matrix(lu.L), k=-1, format="csr")
        dinv = None
        full = strict + sp.eye(strict.shape[0], format="csr")
    strict.sort_indices()
    gptr, order, depth = chain_groups(strict)
    assert gptr[0] == 0 and gptr[-1] == strict.shape[0] and np.diff(gptr).max() <= 32
    # every row of a group after its first depends on the previous row
    for g in range(len(gptr) - 1):
        for r in range(gptr[g] + 1, gptr[g + 1]):
            assert (r - 1) in strict.indices[strict.indptr[r]:strict.indptr[r + 1]]
    dptr, deps = group_dependencies(strict, gptr)
    gid = np.repeat(np.arange(len(gptr) - 1), np.diff(gptr))
    for g in range(len(gptr) - 1):
        rows = range(gptr[g], gptr[g + 1])
        want = set()
        for r in rows:
            cols = strict.indices[strict.indptr[r]:strict.indptr[r + 1]]
            want |= set(gid[cols[cols < gptr[g]]].tolist())
        assert set(deps[dptr[g]:dptr[g + 1]].tolist()) == want
    mptr, minv = group_inverses(strict, gptr, dinv)
    rhs = rng.standard_normal((strict.shape[0], 2))
    y = emulate_group_blocks(strict, dinv, gptr, order, mptr, minv, rhs)
    assert np.abs(full @ y - rhs).max() <= 1e-10 * np.abs(rhs).max()


def test_dense_region_blocks_reproduce_the_factor():
    from paper_2512_23804_b200.linalg import DENSE_BLOCK, chain_groups, dense_blocks, dense_region

    b = build_problem(2, n=16)
    s = steady_system(b)
    a = sp.bmat([[s.mass, None, -s.stiffness[0]], [None, s.beta * s.mass, s.mass],
                 [-s.stiffness[0], s.mass, None]], format="csr")
    lu = spla.splu(sp.csc_matrix(a), diag_pivot_thresh=1.0)
    strict = sp.tril(sp.csr_matrix(lu.L), k=-1, format="csr")
    strict.sort_indices()
    d0, d1 = dense_region(strict)
    assert d1 - d0 >= 128 and (d1 - d0) % DENSE_BLOCK == 0 and d1 == strict.shape[0]
    blk = strict[d0:d1, d0:d1]
    assert blk.nnz >= 0.5 * (d1 - d0) * (d1 - d0 - 1) / 2
    gptr, order, _ = chain_groups(strict, dense=(d0, d1))
    starts = set(gptr.tolist())
    assert all(r in starts for r in range(d0, d1, DENSE_BLOCK))
    assert not any(d0 < r < d1 and (r - d0) % DENSE_BLOCK for r in starts)
    dense = dense_blocks(strict, (d0, d1))
    full = strict.toarray()
    for i in range(1, (d1 - d0) // DENSE_BLOCK):
        r = d0 + DENSE_BLOCK * i
        off = DENSE_BLOCK * DENSE_BLOCK * i * (i - 1) // 2
        got = dense[off:off + DENSE_BLOCK * DENSE_BLOCK * i].reshape(DENSE_BLOCK, DENSE_BLOCK * i)
        assert np.array_equal(got, full[r:r + DENSE_BLOCK, d0:r])


def test_nested_dissection_factor_solves_the_original_system(rng):
    """ordering='nd': SuperLU on P A P^T (NATURAL columns), the outer
    permutation folded into the kernels' row maps — the emulated device solve
    equals A^-1 b, and the triangles are shallower than COLAMD's."""
    from paper_2512_23804_b200.linalg import nested_dissection
    from paper_2512_23804_b200.preconditioners import shifted_lead_terms

    b = build_problem(2, n=24)
    a = shifted_lead_terms(steady_system(b))[0]
    m = int(round(np.sqrt(a.shape[0])))
    p = nested_dissection(m)
    assert np.array_equal(np.sort(p), np.arange(m * m))
    f = sparse_lu(a, ordering="nd")
    lu = f._solver
    outer = f._cache["outer"]
    rhs = rng.standard_normal((a.shape[0], 2))
    want = spla.spsolve(sp.csc_matrix(a), rhs)
    # device row maps: factor row k reads b[outer[iperm_r[k]]], writes x[outer[iperm_c[k]]]
    got = np.zeros_like(rhs)
    got[outer] = emulate_trisolve(lu, rhs[outer])
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    depth_nd = level_schedule(sp.tril(sp.csr_matrix(lu.L), k=-1, format="csr"), lower=True)[1]
    lu_c = sparse_lu(a)._solver
    depth_c = level_schedule(sp.tril(sp.csr_matrix(lu_c.L), k=-1, format="csr"), lower=True)[1]
    assert depth_nd < depth_c
    with pytest.raises(ValueError):
        sparse_lu(sp.identity(12, format="csr"), ordering="nd")
    with pytest.raises(ValueError):
        sparse_lu(a, ordering="amd")
