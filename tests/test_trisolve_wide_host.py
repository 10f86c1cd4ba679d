"""Host-side schedule of the wide-RHS triangular solve (csrc/trisolve_wide.cu,
linalg.wide_tiles): a NumPy emulation of the kernel's tile / segment / slot
bookkeeping on real chain groups must reproduce a dense triangular solve,
every outside entry must be covered exactly once, tiles must respect their
size limits, and every tile's dependencies must be finalised earlier in
ticket order (the deadlock-freedom argument).  CPU only."""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.linalg import solve_triangular

from paper_2512_23804_b200 import linalg


def _strict_lower(n, density, seed, dense_tail=0):
    rng = np.random.default_rng(seed)
    m = sp.random(n, n, density=density, random_state=rng, format="csr")
    m = sp.tril(m, k=-1, format="csr")
    # chains: every row depends on the previous one in runs
    chain = sp.diags(rng.standard_normal(n - 1) * 0.1, -1, shape=(n, n), format="csr")
    m = (m + chain).tocsr()
    if dense_tail:
        blk = np.tril(rng.standard_normal((dense_tail, n)) * 0.01, k=n - dense_tail - 1)
        tail = sp.csr_matrix((n, n))
        tail = sp.vstack([sp.csr_matrix((n - dense_tail, n)), sp.csr_matrix(blk)]).tocsr()
        m = (m + sp.tril(tail, k=-1)).tocsr()
    m.sum_duplicates()
    m.sort_indices()
    return m


def _emulate(strict, gptr, order, dinv, w, b, dense=(0, 0)):
    """The kernel's arithmetic, tile by tile in ticket order."""
    n = strict.shape[0]
    mptr, minv = linalg.group_inverses(strict, gptr, dinv)
    x = np.full_like(b, np.nan)  # unfinished rows poison any early read
    part = np.full((max(1, w["n_slots"]), b.shape[1]), np.nan)
    done_tiles = {}
    ts = w["tile_seg"]
    d0, d1 = dense
    dblk = linalg.dense_blocks(strict, dense) if d1 > d0 else None
    for t in range(w["n_tiles"]):
        g = int(w["tile_group"][t])
        a, bb = int(gptr[g]), int(gptr[g + 1])
        if w["tile_kind"][t] == 1:
            # dense task: all sparse tiles of the group done, earlier region blocks final
            assert done_tiles.get(g, 0) == int(w["group_ntiles"][g])
            bi = (a - d0) // linalg.DENSE_BLOCK
            p_rows = b[a:bb].copy()
            for r in range(a, bb):
                for q in range(w["row_slot_ptr"][r], w["row_slot_ptr"][r + 1]):
                    p_rows[r - a] -= part[w["row_slot"][q]]
            if bi:
                off = linalg.DENSE_BLOCK ** 2 * bi * (bi - 1) // 2
                blk = dblk[off:off + linalg.DENSE_BLOCK * linalg.DENSE_BLOCK * bi].reshape(linalg.DENSE_BLOCK, -1)
                p_rows -= blk @ x[d0:a]
            g_n = bb - a
            mi = minv[mptr[g]:mptr[g] + g_n * g_n].reshape(g_n, g_n)
            x[a:bb] = mi @ p_rows
            continue
        sp_ = []
        for s in range(ts[t], ts[t + 1]):
            e0, e1 = w["seg_e0"][s], w["seg_e1"][s]
            cols = strict.indices[e0:e1]
            sp_.append(strict.data[e0:e1] @ x[cols])
        nt = int(w["group_ntiles"][g])
        is_dense = d1 > d0 and d0 <= a < d1
        if w["tile_kind"][t] == 2:
            # designated finaliser: the group's other tiles are done
            assert done_tiles.get(g, 0) == nt - 1
            p_rows = b[a:bb].copy()
            for s in range(ts[t], ts[t + 1]):
                p_rows[w["seg_row"][s] - a] -= sp_[s - ts[t]]
            for r in range(a, bb):
                for q in range(w["row_slot_ptr"][r], w["row_slot_ptr"][r + 1]):
                    p_rows[r - a] -= part[w["row_slot"][q]]
        elif nt > 1 or is_dense:
            acc = None
            for s in range(ts[t], ts[t + 1]):
                v = sp_[s - ts[t]]
                acc = v if acc is None else acc + v
                if s + 1 == ts[t + 1] or w["seg_slot"][s + 1] != w["seg_slot"][s]:
                    part[w["seg_slot"][s]] = acc
                    acc = None
            done_tiles[g] = done_tiles.get(g, 0) + 1
            if done_tiles[g] < nt or is_dense:
                continue
            p_rows = b[a:bb].copy()
            for r in range(a, bb):
                for q in range(w["row_slot_ptr"][r], w["row_slot_ptr"][r + 1]):
                    p_rows[r - a] -= part[w["row_slot"][q]]
        else:
            p_rows = b[a:bb].copy()
            for s in range(ts[t], ts[t + 1]):
                p_rows[w["seg_row"][s] - a] -= sp_[s - ts[t]]
        g_n = bb - a
        mi = minv[mptr[g]:mptr[g] + g_n * g_n].reshape(g_n, g_n)
        x[a:bb] = mi @ p_rows
    return x


def _check(strict, dinv, dense=(0, 0)):
    gptr, order, _ = linalg.chain_groups(strict, dense=dense)
    w = linalg.wide_tiles(strict, gptr, order, dense)
    n = strict.shape[0]
    # coverage: every outside entry exactly once, in-group / in-region entries never
    gid = np.repeat(np.arange(len(gptr) - 1), np.diff(gptr))
    row_of = np.repeat(np.arange(n), np.diff(strict.indptr))
    left = gptr[gid[row_of]]
    if dense[1] > dense[0]:
        left = np.where((row_of >= dense[0]) & (row_of < dense[1]), dense[0], left)
    outside = strict.indices < left
    hit = np.zeros(strict.nnz, np.int64)
    for e0, e1 in zip(w["seg_e0"], w["seg_e1"]):
        assert 1 <= e1 - e0 <= linalg.WIDE_SEG
        hit[e0:e1] += 1
    assert np.array_equal(hit, outside.astype(np.int64))
    ts = w["tile_seg"]
    assert np.all(np.diff(ts) <= linalg.WIDE_TILE_SEGS)
    # dependencies finalised by earlier tiles (groups in topological order)
    first_tile = {}
    last_tile = {}
    for t, g in enumerate(w["tile_group"]):
        first_tile.setdefault(int(g), t)
        last_tile[int(g)] = t
    for t in range(w["n_tiles"]):
        for d in w["dep"][w["dep_ptr"][t]:w["dep_ptr"][t + 1]]:
            assert last_tile[int(d)] < first_tile[int(w["tile_group"][t])]
    rng = np.random.default_rng(3)
    b = rng.standard_normal((n, 5))
    x = _emulate(strict, gptr, order, dinv, w, b, dense)
    full = strict.toarray()
    full[np.arange(n), np.arange(n)] = 1.0 if dinv is None else 1.0 / np.asarray(dinv)
    want = solve_triangular(full, b, lower=True)
    assert np.abs(x - want).max() <= 1e-11 * np.abs(want).max()
    return w


def test_wide_tiles_unit_lower():
    strict = _strict_lower(300, 0.05, 1)
    w = _check(strict, None)
    assert w["n_tiles"] >= 1


def test_wide_tiles_heavy_rows_split_over_tiles():
    # dense trailing rows: > 256 outside entries per group, several tiles,
    # part slots, the finalising tile sums them in tile order
    strict = _strict_lower(400, 0.02, 2, dense_tail=96)
    dinv = 1.0 / (1.0 + np.random.default_rng(5).random(400))
    w = _check(strict, dinv)
    assert int(w["group_ntiles"].max()) > 1 and w["n_slots"] > 0


def test_wide_tiles_with_dense_region_groups():
    strict = _strict_lower(512, 0.01, 4, dense_tail=160)
    dense = linalg.dense_region(strict)
    assert dense[1] - dense[0] >= 64
    w = _check(strict, None, dense=dense)
    assert int(np.sum(w["tile_kind"] == 1)) == (dense[1] - dense[0]) // linalg.DENSE_BLOCK


# ---- column-panel form (linalg.wide_panels, trsv_wide<PANEL>) -----------------

def _emulate_panels(strict, gptr, dinv, w, b, dense=(0, 0)):
    """The PANEL kernel's arithmetic, tile by tile in ticket order."""
    mptr, minv = linalg.group_inverses(strict, gptr, dinv)
    x = np.full_like(b, np.nan)
    part = np.full((max(1, w["n_slots"]), b.shape[1]), np.nan)
    done_tiles = {}
    tp = w["tile_seg"]
    d0, d1 = dense
    dblk = linalg.dense_blocks(strict, dense) if d1 > d0 else None
    pc = w["pcol"].reshape(-1, linalg.PANEL_COLS)
    pv = w["pval"].reshape(-1, linalg.PANEL_COLS, linalg.PANEL_COLS)

    def minus_slots(p_rows, a, bb):
        for r in range(a, bb):
            for q in range(w["row_slot_ptr"][r], w["row_slot_ptr"][r + 1]):
                p_rows[r - a] -= part[w["row_slot"][q]]

    for t in range(w["n_tiles"]):
        g = int(w["tile_group"][t])
        a, bb = int(gptr[g]), int(gptr[g + 1])
        g_n = bb - a
        nt = int(w["group_ntiles"][g])
        is_dense = d1 > d0 and d0 <= a < d1
        kind = int(w["tile_kind"][t])
        if kind == 1:
            assert done_tiles.get(g, 0) == nt
            bi = (a - d0) // linalg.DENSE_BLOCK
            p_rows = b[a:bb].copy()
            minus_slots(p_rows, a, bb)
            if bi:
                off = linalg.DENSE_BLOCK ** 2 * bi * (bi - 1) // 2
                blk = dblk[off:off + linalg.DENSE_BLOCK * linalg.DENSE_BLOCK * bi].reshape(linalg.DENSE_BLOCK, -1)
                p_rows -= blk @ x[d0:a]
        else:
            acc = np.zeros((linalg.PANEL_COLS, b.shape[1]))
            for pi in range(tp[t], tp[t + 1]):
                xs = x[pc[pi]]
                assert np.all(np.isfinite(xs)), "panel reads an unfinished row"
                acc += pv[pi] @ xs
            assert np.all(acc[g_n:] == 0.0)
            if kind == 2 or (nt == 1 and not is_dense):
                p_rows = b[a:bb] - acc[:g_n]
                if kind == 2:
                    assert done_tiles.get(g, 0) == nt - 1
                    minus_slots(p_rows, a, bb)
            else:
                s0 = int(w["tile_slot"][t])
                assert s0 >= 0
                part[s0:s0 + g_n] = acc[:g_n]
                done_tiles[g] = done_tiles.get(g, 0) + 1
                continue
        mi = minv[mptr[g]:mptr[g] + g_n * g_n].reshape(g_n, g_n)
        x[a:bb] = mi @ p_rows
    return x


def _check_panels(strict, dinv, dense=(0, 0), panels_per_tile=2):
    gptr, order, _ = linalg.chain_groups(strict, dense=dense)
    w = linalg.wide_panels(strict, gptr, order, dense, panels_per_tile=panels_per_tile)
    n = strict.shape[0]
    # the panels hold every outside entry exactly once and nothing else
    gid = np.repeat(np.arange(len(gptr) - 1), np.diff(gptr))
    row_of = np.repeat(np.arange(n), np.diff(strict.indptr))
    left = gptr[gid[row_of]]
    if dense[1] > dense[0]:
        left = np.where((row_of >= dense[0]) & (row_of < dense[1]), dense[0], left)
    outside = strict.indices < left
    want_sum = sp.csr_matrix((strict.data[outside], (row_of[outside], strict.indices[outside])), shape=(n, n))
    rec = sp.lil_matrix((n, n))
    pc = w["pcol"].reshape(-1, linalg.PANEL_COLS)
    pv = w["pval"].reshape(-1, linalg.PANEL_COLS, linalg.PANEL_COLS)
    tp = w["tile_seg"]
    assert np.all(np.diff(tp) <= panels_per_tile)
    for t in range(w["n_tiles"]):
        a = int(gptr[int(w["tile_group"][t])])
        for pi in range(tp[t], tp[t + 1]):
            r, k = np.nonzero(pv[pi])
            for rr, kk in zip(r, k):
                assert rec[a + rr, pc[pi, kk]] == 0.0
                rec[a + rr, pc[pi, kk]] = pv[pi, rr, kk]
    assert abs(rec.tocsr() - want_sum).max() == 0.0
    # every group is finalised by exactly one task, dependencies by earlier tickets
    first_tile, last_tile = {}, {}
    for t, g in enumerate(w["tile_group"]):
        first_tile.setdefault(int(g), t)
        last_tile[int(g)] = t
    assert len(first_tile) == len(gptr) - 1
    for t in range(w["n_tiles"]):
        for d in w["dep"][w["dep_ptr"][t]:w["dep_ptr"][t + 1]]:
            assert last_tile[int(d)] < first_tile[int(w["tile_group"][t])]
    rng = np.random.default_rng(3)
    b = rng.standard_normal((n, 5))
    x = _emulate_panels(strict, gptr, dinv, w, b, dense)
    full = strict.toarray()
    full[np.arange(n), np.arange(n)] = 1.0 if dinv is None else 1.0 / np.asarray(dinv)
    want = solve_triangular(full, b, lower=True)
    assert np.abs(x - want).max() <= 1e-11 * np.abs(want).max()
    return w


def test_wide_panels_unit_lower():
    w = _check_panels(_strict_lower(300, 0.05, 1), None)
    assert w["n_panels"] >= 1


def test_wide_panels_heavy_groups_split_over_tiles():
    strict = _strict_lower(400, 0.02, 2, dense_tail=96)
    dinv = 1.0 / (1.0 + np.random.default_rng(5).random(400))
    w = _check_panels(strict, dinv)
    assert int(w["group_ntiles"].max()) > 1 and w["n_slots"] > 0


def test_wide_panels_with_dense_region_groups():
    strict = _strict_lower(512, 0.01, 4, dense_tail=160)
    dense = linalg.dense_region(strict)
    w = _check_panels(strict, None, dense=dense)
    assert int(np.sum(w["tile_kind"] == 1)) == (dense[1] - dense[0]) // linalg.DENSE_BLOCK


def test_wide_panels_group_without_outside_entries_gets_a_tile():
    strict = sp.csr_matrix(np.tril(np.ones((40, 40)), k=-1) * 0.01)  # one chain: later groups depend on earlier
    strict = sp.block_diag([strict, sp.csr_matrix((8, 8))], format="csr")  # 8 isolated rows
    _check_panels(strict, None)
