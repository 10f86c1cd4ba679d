"""Schedules compiled by program.py, executed by a NumPy emulation of the
device kernels, against dense products (CPU only)."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2512_23804_b200.basis import build_triple_products, enumerate_multi_indices, level_partition
from paper_2512_23804_b200.program import compile_program, compile_program9, coupling_from_csr, emulate, emulate9


def _system(rng, n=12, m=3, p=3, deg=1, family="legendre"):
    b = enumerate_multi_indices(m, p)
    tp = build_triple_products(b, enumerate_multi_indices(m, deg), family=family)
    pat = sp.random(n, n, density=0.4, random_state=1, format="csr") + sp.eye(n, format="csr")
    pat.data[:] = 1.0
    pat.sort_indices()
    mats = []
    for _ in range(tp.n_terms + 1):
        a = pat.copy()
        a.data = rng.standard_normal(a.nnz)
        mats.append(a)
    return b, tp, pat, mats


def _check(rng, cps, widths, inputs, inits, alpha, beta, mats, pat, expect):
    for mode in ("uniform", "packed"):
        for budget in (6144, 96):
            prog = compile_program(cps, widths, mode=mode, budget_slots=budget)
            outs = emulate(prog, pat.indptr, pat.indices, [m.data for m in mats], inputs, inits, alpha, beta)
            for o, e in zip(outs, expect):
                assert np.abs(o - e).max() <= 1e-12 * max(1.0, np.abs(e).max())
    prog9 = compile_program9(cps, widths)
    outs = emulate9(prog9, mats, inputs, inits, alpha, beta)
    for o, e in zip(outs, expect):
        assert np.abs(o - e).max() <= 1e-12 * max(1.0, np.abs(e).max())


def test_full_kron_program(rng):
    b, tp, pat, mats = _system(rng)
    n_xi = b.size
    x = rng.standard_normal((pat.shape[0], n_xi))
    cps = [coupling_from_csr(0, 0, t, tp.matrices[t], (0, n_xi), (0, n_xi)) for t in range(tp.n_terms)]
    expect = sum(mats[t] @ x @ tp.matrices[t].toarray() for t in range(tp.n_terms))
    _check(rng, cps, (n_xi,), [x], [None], [1.0], [0.0], mats, pat, [expect])


def test_sliced_level_programs_with_init(rng):
    b, tp, pat, mats = _system(rng, m=2, p=3)
    n_xi = b.size
    part = level_partition(b)
    x = rng.standard_normal((pat.shape[0], n_xi))
    r = rng.standard_normal((pat.shape[0], n_xi))
    for lo, hi in part.ranges():
        for srcs in ([(0, lo)], [(0, lo), (hi, n_xi)]):
            cps = []
            expect = r[:, lo:hi].copy()
            for t in range(1, tp.n_terms):
                h = tp.matrices[t].tocsr()
                for (a, bb) in srcs:
                    cps.append(coupling_from_csr(0, 0, t, h, (a, bb), (lo, hi), -1.0))
                    if bb > a:
                        expect -= mats[t] @ x[:, a:bb] @ h[a:bb, lo:hi].toarray()
            _check(rng, cps, (hi - lo,), [x], [r[:, lo:hi]], [1.0], [1.0], mats, pat, [expect])


def test_three_input_kkt_like_program(rng):
    b, tp, pat, mats = _system(rng, m=2, p=2, deg=2, family="hermite")
    n_xi = b.size
    T = tp.n_terms
    n = pat.shape[0]
    ys = [rng.standard_normal((n, n_xi)) for _ in range(3)]
    wdiag = sp.diags(1.0 + np.arange(n_xi), format="csr")
    eye = sp.identity(n_xi, format="csr")
    m = T  # mass slice index
    cps = [coupling_from_csr(0, 0, m, wdiag, (0, n_xi), (0, n_xi))]
    for t in range(T):
        cps.append(coupling_from_csr(2, 0, t, tp.matrices[t], (0, n_xi), (0, n_xi), -1.0))
        cps.append(coupling_from_csr(0, 2, t, tp.matrices[t], (0, n_xi), (0, n_xi), -1.0))
    cps.append(coupling_from_csr(1, 1, m, eye, (0, n_xi), (0, n_xi), 0.5))
    cps.append(coupling_from_csr(2, 1, m, eye, (0, n_xi), (0, n_xi), 1.0))
    cps.append(coupling_from_csr(1, 2, m, eye, (0, n_xi), (0, n_xi), 1.0))
    A = lambda v: sum(mats[t] @ v @ tp.matrices[t].toarray() for t in range(T))
    M = mats[m]
    expect = [M @ ys[0] @ wdiag.toarray() - A(ys[2]), 0.5 * M @ ys[1] + M @ ys[2], -A(ys[0]) + M @ ys[1]]
    _check(rng, cps, (n_xi,) * 3, ys, [None] * 3, [1.0] * 3, [0.0] * 3, mats, pat, expect)


def test_empty_program_copies_init(rng):
    r = rng.standard_normal((6, 4))
    prog = compile_program([], (4,))
    assert prog.n_groups == 0 and prog.n_phases == 0
    out = emulate(prog, np.arange(7), np.arange(6), [np.ones(6)], [r], [r], [1.0], [2.0])[0]
    assert np.array_equal(out, 2.0 * r)
    p9 = compile_program9([], (4,))
    assert p9.n_groups == 0
    out9 = emulate9(p9, [sp.identity(6, format="csr")], [r], [r], [1.0], [2.0])[0]
    assert np.array_equal(out9, 2.0 * r)


def test_program_validation():
    with pytest.raises(ValueError):
        compile_program([], ())
    with pytest.raises(ValueError):
        compile_program([], (1,) * 5)


def test_assign_rows_keeps_entries_and_spreads_banks(rng):
    from paper_2512_23804_b200.program import _assign_rows

    zero_of_bank = {b: 10_000 + b for b in range(16)}
    lists = []
    for lane in range(32):
        k = int(rng.integers(0, 9))
        lists.append([(int(p), int(p) % 16) for p in rng.choice(5000, size=k, replace=False)])
    rows = _assign_rows(lists, zero_of_bank)
    assert len(rows) == max(len(x) for x in lists)
    for lane in range(32):
        got = sorted(int(v) for v in rows[:, lane] if v < 10_000)
        assert got == sorted(p for p, _ in lists[lane])
    # per row and half-warp, no more repeated bank pairs than forced
    waves = 0
    for r in rows:
        for h in (r[:16], r[16:]):
            waves += np.bincount(np.unique(h) % 16, minlength=16).max()
    bound = 0
    for half in (range(16), range(16, 32)):
        load = np.zeros(16, int)
        for ln in half:
            for p, b in lists[ln]:
                load[b] += 1
        bound += max(len(rows), load.max())
    assert waves <= bound + len(rows)  # the per-row matching is near the model bound


def test_stencil9_gather_layout_covers_every_entry(rng):
    """Every (output, product) coupling appears exactly once in the packed
    gather (and the emulation matches dense products)."""
    b, tp, pat, mats = _system(rng, n=10, m=3, p=3)
    hs = tp.matrices
    n_xi = hs[0].shape[0]
    cps = [coupling_from_csr(0, 0, t, hs[t].tocsr(), (0, n_xi), (0, n_xi), 1.0) for t in range(len(hs))]
    p9 = compile_program9(cps, (n_xi,), n_slices_hint=len(hs))
    assert p9.stats["gather_rows"] >= max(int(h.getnnz(axis=0).max()) for h in hs)
    x = rng.standard_normal((10, n_xi))
    want = sum(mats[t] @ x @ hs[t].toarray() for t in range(len(hs)))
    assert p9.n_slices == len(hs)
    got = emulate9(p9, mats[: len(hs)], [x], [None], [1.0], [0.0])[0]
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
