"""Host compiler for Galerkin coupling programs (the schedule the fused
device kernel `program_kernel` in csrc/galerkin.cu executes).

A *program* is a set of couplings

    out_o[:, k] += c * (A_t V_s)[:, l]        for entries (s, o, t, l, k, c)

which covers every hot-path product of the reference:

* kron_apply              operators.py:88-96  (s=o=0, t<n_t, H_t entries)
* kron_apply_sliced       operators.py:99-126 (entries restricted to src x dst)
* HGS._cross_product      preconditioners.py:132-144 (t>=1, coefficient -h)
* hGSoc._level_rhs        preconditioners.py:386-409 (3 inputs, 3 outputs)
* steady_kkt_apply        operators.py:181-194 (mass as an extra slice)

Compilation:
1. every distinct product (s, l, t) becomes one stencil dot U_(s,l,t);
2. products sharing an input column (s, l) form an *item*; an item lives in
   one lane so the nine neighbour values V_s[j, l] stay in registers while
   all its t are evaluated;
3. items are packed 32 to a *group* (one warp); a group runs a list of
   *steps* and at each step lane lambda evaluates the term step_term[q, lambda]
   (-1 = idle).  "uniform" schedules give every lane the same t at a step
   (the coefficient loads become warp broadcasts) at the price of idle lanes;
   "packed" schedules give each lane its own term list (no idle lanes,
   per-lane coefficient loads) — better when there are hundreds of terms;
4. groups are cut into *phases* whose U values fit the shared-memory budget;
5. the sparse H couplings become, per phase, a CSR gather list over output
   columns reading U from shared memory.
"""

from __future__ import annotations

from dataclasses import dataclass, field
import os

import numpy as np

__all__ = ["Coupling", "HostProgram", "compile_program", "coupling_from_csr"]


@dataclass(frozen=True)
class Coupling:
    """Entries out_o[:, cols] += vals * (A_t V_s)[:, rows]."""

    s: int
    o: int
    t: int
    rows: np.ndarray  # input column l (relative to the input view)
    cols: np.ndarray  # output column k (relative to the output view)
    vals: np.ndarray


def coupling_from_csr(s, o, t, h, row_range, col_range, scale=1.0) -> Coupling | None:
    """Entries of h[rlo:rhi, clo:chi] as a coupling (rows offset by rlo: they
    index the full input; cols relative to clo: they index the output view).
    Returns None when the slice is empty (the reference skips those terms,
    operators.py:124, preconditioners.py:142,369,382)."""
    rlo, rhi = row_range
    clo, chi = col_range
    if rlo >= rhi or clo >= chi:
        return None
    sub = h[rlo:rhi, clo:chi].tocoo()
    keep = sub.data != 0.0
    if not np.any(keep):
        return None
    return Coupling(
        s=s,
        o=o,
        t=t,
        rows=sub.row[keep].astype(np.int64) + rlo,
        cols=sub.col[keep].astype(np.int64),
        vals=scale * sub.data[keep],
    )


@dataclass
class HostProgram:
    n_groups: int
    n_phases: int
    n_out_cols: int
    max_phase_slots: int
    lane_item: np.ndarray
    group_step0: np.ndarray
    step_term: np.ndarray
    phase_group0: np.ndarray
    gather_ptr: np.ndarray
    gather_slot: np.ndarray
    gather_coef: np.ndarray
    out_col: np.ndarray
    out_widths: tuple[int, ...]
    stats: dict = field(default_factory=dict)


def _schedule_uniform(item_terms: list[np.ndarray], order: np.ndarray):
    groups = []
    for g0 in range(0, len(order), 32):
        members = order[g0 : g0 + 32]
        union = np.unique(np.concatenate([item_terms[i] for i in members]))
        groups.append((members, union))
    return groups


def _uniform_cost(groups) -> int:
    return sum(len(u) for _, u in groups)


def _best_uniform(item_terms: list[np.ndarray]):
    n = len(item_terms)
    keys_lex = sorted(range(n), key=lambda i: tuple(item_terms[i]))
    keys_len = sorted(range(n), key=lambda i: (-len(item_terms[i]), tuple(item_terms[i])))
    best = None
    for order in (np.array(keys_lex, dtype=np.int64), np.array(keys_len, dtype=np.int64)):
        groups = _schedule_uniform(item_terms, order)
        cost = _uniform_cost(groups)
        if best is None or cost < best[0]:
            best = (cost, groups)
    return best


def compile_program(
    couplings: list[Coupling],
    out_widths: tuple[int, ...] | list[int],
    *,
    n_inputs: int | None = None,
    budget_slots: int = 6144,
    mode: str = "auto",
    packed_chunk: int = 16,
) -> HostProgram:
    out_widths = tuple(int(w) for w in out_widths)
    if not out_widths or len(out_widths) > 4:
        raise ValueError("a program has 1..4 outputs")
    couplings = [c for c in couplings if c is not None and len(c.rows)]
    if n_inputs is None:
        n_inputs = 1 + max((c.s for c in couplings), default=0)
    if n_inputs > 4:
        raise ValueError("a program has at most 4 inputs")
    out_off = np.concatenate([[0], np.cumsum(out_widths)]).astype(np.int64)
    n_out_cols = int(out_off[-1])

    # ---- 1. distinct products (s, l, t) and gather entries ------------------
    if couplings:
        s_arr = np.concatenate([np.full(len(c.rows), c.s, np.int64) for c in couplings])
        t_arr = np.concatenate([np.full(len(c.rows), c.t, np.int64) for c in couplings])
        l_arr = np.concatenate([np.asarray(c.rows, np.int64) for c in couplings])
        o_arr = np.concatenate([np.full(len(c.rows), c.o, np.int64) for c in couplings])
        k_arr = np.concatenate([np.asarray(c.cols, np.int64) for c in couplings])
        v_arr = np.concatenate([np.asarray(c.vals, np.float64) for c in couplings])
    else:
        s_arr = t_arr = l_arr = o_arr = k_arr = np.zeros(0, np.int64)
        v_arr = np.zeros(0)
    if np.any(k_arr < 0) or np.any(k_arr >= np.asarray(out_widths)[o_arr] if len(o_arr) else False):
        raise ValueError("coupling column outside its output view")
    if np.any(l_arr < 0) or np.any(l_arr >= (1 << 24)):
        raise ValueError("input column out of range")
    big_t = int(t_arr.max()) + 1 if len(t_arr) else 1
    big_l = int(l_arr.max()) + 1 if len(l_arr) else 1
    pair_key = (s_arr * big_l + l_arr) * big_t + t_arr
    uniq, pair_of_entry = np.unique(pair_key, return_inverse=True)
    p_t = uniq % big_t
    p_item_key = uniq // big_t  # (s, l)
    item_keys, item_of_pair = np.unique(p_item_key, return_inverse=True)
    n_items = len(item_keys)
    item_terms = [np.zeros(0, np.int64)] * n_items
    if n_items:
        order_pairs = np.argsort(item_of_pair, kind="stable")
        splits = np.cumsum(np.bincount(item_of_pair, minlength=n_items))[:-1]
        item_pair_lists = np.split(order_pairs, splits)
        item_terms = [p_t[pl] for pl in item_pair_lists]
    else:
        item_pair_lists = []

    # ---- 2./3. items -> groups -> steps ---------------------------------------
    groups = []  # list of (lane_items[list of item or -1 per lane], steps[q][lane] -> t or -1)
    chosen = "none"
    if n_items:
        uni_cost, uni_groups = _best_uniform(item_terms)
        # packed: split long term lists, pack by length
        sub_items = []
        for i, terms in enumerate(item_terms):
            for a in range(0, len(terms), packed_chunk):
                sub_items.append((i, terms[a : a + packed_chunk]))
        sub_items.sort(key=lambda it: -len(it[1]))
        packed_groups = [sub_items[g : g + 32] for g in range(0, len(sub_items), 32)]
        packed_cost = sum(len(g[0][1]) for g in packed_groups)
        use_packed = mode == "packed" or (mode == "auto" and 2 * packed_cost < uni_cost)
        if use_packed:
            chosen = "packed"
            for g in packed_groups:
                nsteps = len(g[0][1])
                lanes = [it[0] for it in g] + [-1] * (32 - len(g))
                steps = -np.ones((nsteps, 32), np.int64)
                # each lane's terms may run in any order: at every step pick,
                # lane by lane, the remaining term whose coefficients sit in the
                # least-used shared-memory bank pair (the row block is staged
                # as t*9 + jj doubles: bank pair (9 t) mod 16), so the per-lane
                # coefficient loads of a step conflict less (config 3: 5.9 ->
                # 3.0 wavefronts per load on average, ideal 2)
                remaining = [list(terms) for _, terms in g]
                for q in range(nsteps):
                    used = np.zeros(16, np.int64)
                    for lane, rem in enumerate(remaining):
                        if not rem:
                            continue
                        k = min(range(len(rem)), key=lambda i: (used[(rem[i] * 9) % 16], i))
                        t = rem.pop(k)
                        steps[q, lane] = t
                        used[(t * 9) % 16] += 1
                groups.append((lanes, steps))
        else:
            chosen = "uniform"
            for members, union in uni_groups:
                lanes = list(members) + [-1] * (32 - len(members))
                steps = -np.ones((len(union), 32), np.int64)
                for lane, it in enumerate(members):
                    mask = np.isin(union, item_terms[it])
                    steps[mask, lane] = union[mask]
                groups.append((lanes, steps))

    # split groups whose steps alone exceed the phase budget
    max_steps = max(1, budget_slots // 32)
    split_groups = []
    for lanes, steps in groups:
        for a in range(0, len(steps), max_steps):
            split_groups.append((lanes, steps[a : a + max_steps]))
    groups = split_groups

    # ---- 4. phases -----------------------------------------------------------
    phase_group0 = [0]
    group_step0 = [0]
    acc = 0
    for gi, (_, steps) in enumerate(groups):
        if acc + len(steps) > max_steps and acc > 0:
            phase_group0.append(gi)
            acc = 0
        acc += len(steps)
        group_step0.append(group_step0[-1] + len(steps))
    if groups:
        phase_group0.append(len(groups))
    n_phases = len(phase_group0) - 1 if groups else 0
    n_groups = len(groups)
    total_steps = group_step0[-1]

    lane_item = -np.ones(max(n_groups, 0) * 32, np.int64)
    step_term = -np.ones((total_steps, 32), np.int64)
    # pair -> (phase, slot)
    n_pairs = len(uniq)
    pair_phase = -np.ones(n_pairs, np.int64)
    pair_slot = -np.ones(n_pairs, np.int64)
    # per item: term -> pair id
    item_term_pair = []
    for i in range(n_items):
        item_term_pair.append(dict(zip(item_terms[i].tolist(), item_pair_lists[i].tolist())))
    ph = 0
    for gi, (lanes, steps) in enumerate(groups):
        while ph + 1 < len(phase_group0) and gi >= phase_group0[ph + 1]:
            ph += 1
        qbase = group_step0[phase_group0[ph]]
        q0 = group_step0[gi]
        step_term[q0 : q0 + len(steps)] = steps
        for lane, it in enumerate(lanes):
            if it < 0:
                continue
            key = int(item_keys[it])
            s_i, l_i = divmod(key, big_l)
            lane_item[gi * 32 + lane] = (s_i << 24) | l_i
            col = steps[:, lane]
            for qq in np.flatnonzero(col >= 0):
                pid = item_term_pair[it][int(col[qq])]
                if pair_phase[pid] >= 0:
                    raise AssertionError("product scheduled twice")
                pair_phase[pid] = ph
                pair_slot[pid] = (q0 + qq - qbase) * 32 + lane
    if n_pairs and np.any(pair_phase < 0):
        raise AssertionError("unscheduled product")

    # ---- 5. gather lists -----------------------------------------------------
    n_ent = len(v_arr)
    c_arr = out_off[o_arr] + k_arr if n_ent else np.zeros(0, np.int64)
    e_phase = pair_phase[pair_of_entry] if n_ent else np.zeros(0, np.int64)
    e_slot = pair_slot[pair_of_entry] if n_ent else np.zeros(0, np.int64)
    e_t = t_arr
    ordr = np.lexsort((l_arr, e_t, c_arr, e_phase)) if n_ent else np.zeros(0, np.int64)
    n_ptr = max(n_phases, 0) * n_out_cols
    counts = np.bincount(e_phase * n_out_cols + c_arr, minlength=n_ptr) if n_ent else np.zeros(n_ptr, np.int64)
    gather_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    gather_slot = e_slot[ordr]
    gather_coef = v_arr[ordr]
    o_of_c = np.repeat(np.arange(len(out_widths)), out_widths)
    k_of_c = np.concatenate([np.arange(w) for w in out_widths]) if n_out_cols else np.zeros(0, np.int64)
    out_col = (o_of_c << 24) | k_of_c

    max_slots = 0
    for p in range(n_phases):
        q_lo = group_step0[phase_group0[p]]
        q_hi = group_step0[phase_group0[p + 1]]
        max_slots = max(max_slots, (q_hi - q_lo) * 32)

    useful = n_pairs
    executed = total_steps * 32
    stats = {
        "mode": chosen,
        "n_products": int(useful),
        "n_items": int(n_items),
        "n_groups": int(n_groups),
        "n_steps": int(total_steps),
        "lane_efficiency": float(useful / executed) if executed else 1.0,
        "n_gather": int(n_ent),
    }
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
    return HostProgram(
        n_groups=n_groups,
        n_phases=n_phases,
        n_out_cols=n_out_cols,
        max_phase_slots=int(max_slots),
        lane_item=i32(lane_item),
        group_step0=i32(group_step0),
        step_term=i32(step_term.reshape(-1)),
        phase_group0=i32(phase_group0 if n_phases else [0]),
        gather_ptr=i32(gather_ptr),
        gather_slot=i32(gather_slot),
        gather_coef=np.ascontiguousarray(gather_coef, dtype=np.float64),
        out_col=i32(out_col),
        out_widths=out_widths,
        stats=stats,
    )


def emulate(prog: HostProgram, pattern_rowptr, pattern_colind, slice_vals_std, inputs, inits, alpha, beta):
    """NumPy emulation of program_kernel (test-only helper for the schedule;
    slice_vals_std[t] is the CSR data array of slice t on the pattern)."""
    n_rows = len(pattern_rowptr) - 1
    import scipy.sparse as sp

    mats = [sp.csr_matrix((v, pattern_colind, pattern_rowptr), shape=(n_rows, inputs[0].shape[0])) for v in slice_vals_std]
    outs = []
    acc = np.zeros((n_rows, prog.n_out_cols))
    steps = prog.step_term.reshape(-1, 32)
    for p in range(prog.n_phases):
        ub = np.zeros((n_rows, prog.max_phase_slots))
        g0, g1 = prog.phase_group0[p], prog.phase_group0[p + 1]
        qbase = prog.group_step0[g0]
        for g in range(g0, g1):
            for lane in range(32):
                item = prog.lane_item[g * 32 + lane]
                if item < 0:
                    continue
                s, l = item >> 24, item & 0xFFFFFF
                for q in range(prog.group_step0[g], prog.group_step0[g + 1]):
                    t = steps[q, lane]
                    if t >= 0:
                        ub[:, (q - qbase) * 32 + lane] = mats[t] @ inputs[s][:, l]
        for c in range(prog.n_out_cols):
            e0, e1 = prog.gather_ptr[p * prog.n_out_cols + c], prog.gather_ptr[p * prog.n_out_cols + c + 1]
            for e in range(e0, e1):
                acc[:, c] += prog.gather_coef[e] * ub[:, prog.gather_slot[e]]
    off = 0
    for o, w in enumerate(prog.out_widths):
        y = alpha[o] * acc[:, off : off + w]
        if inits[o] is not None:
            y = y + beta[o] * inits[o]
        outs.append(y)
        off += w
    return outs


@dataclass
class HostProgram9:
    """Contiguous-group uniform schedule for the 9-point fast path
    (csrc/stencil9.cu; layout documented in include/sgkkt_b200.h)."""

    n_groups: int
    n_steps: int
    n_ubuf: int
    n_out_cols: int
    n_coef: int
    n_gather: int
    group_info: np.ndarray
    step_rec: np.ndarray
    coef_tab: np.ndarray
    gather_ptr: np.ndarray
    gather_ent: np.ndarray
    out_col: np.ndarray
    out_widths: tuple[int, ...]
    stats: dict = field(default_factory=dict)
    n_slices: int = 0
    warps: int = 1  # CTA warps the gather layout assumes (chunk c -> warp c % warps)


# 4 column slots x 32 lanes (SGKKT_S9_KC selects another slot count; the
# library must be built with the same -DSGK_S9_KC)
GROUP_COLS = 32 * int(os.environ.get("SGKKT_S9_KC", "4"))


# up to 16 warps (one 512-thread CTA per SM) so programs with 9..16 column
# groups keep every group resident; SGKKT_S9_BIG=0 caps CTAs at 8 warps
S9_BIG = os.environ.get("SGKKT_S9_BIG", "1") != "0"


def stencil9_warps(n_groups: int, n_chunks: int) -> int:
    """Warps per CTA for stencil9_kernel: one per column group (resident V
    registers) and at most 16 gather chunks per warp; 8 at most, 16 for
    programs with 9..16 groups."""
    # gather-heavy programs (few column groups, many output chunks) get up to
    # 8 warps so each gathers <= 4 chunks
    w = max(1, n_groups, -(-n_chunks // 16), min(8, -(-n_chunks // 4)))
    if S9_BIG and 8 < n_groups <= 16:
        return min(16, w)
    return min(8, w)
# bank-layout local search budget per program (deterministic; off by default:
# cfg4 matvec 1.725 ms with it vs 1.728 ms without, and it costs ~3 s/program)
SEARCH_MOVES = int(os.environ.get("SGKKT_S9_SEARCH_MOVES", "0"))


def _ubuf_base(n_coef: int, n_slices: int) -> int:
    """Byte offset of ubuf in stencil9_kernel's dynamic shared memory."""
    a16 = lambda x: (x + 15) & ~15
    return a16(a16(a16(8 * n_coef) + 2 * 8 * n_slices * 10) + 2 * 16 * 4)


def _class_layout(counts, out_off, n_cls):
    """Output positions: each output's columns sorted by their per-class entry
    counts (so a 32-lane chunk has similar counts per class), padded to whole
    chunks (a chunk never spans two outputs).  Returns (col_at_pos, pos_of_col)."""
    col_at_pos = []
    for o in range(len(out_off) - 1):
        cols = np.arange(out_off[o], out_off[o + 1])
        if len(cols):
            keys = tuple(-counts[cols, c] for c in range(n_cls))
            cols = cols[np.lexsort(keys)]
        pad = (-len(cols)) % 32
        col_at_pos.extend(cols.tolist() + [-1] * pad)
    col_at_pos = np.array(col_at_pos, dtype=np.int64)
    pos_of_col = np.full(int(out_off[-1]), -1, np.int64)
    valid = col_at_pos >= 0
    pos_of_col[col_at_pos[valid]] = np.nonzero(valid)[0]
    return col_at_pos, pos_of_col


class _BankSearch:
    """Deterministic local search over (per-step slot swizzle, output position
    permutation) minimising the modelled U-gather shared-memory wavefronts
    sum_cells max(rows(cell), max bank-pair load(cell)), cell = (chunk, class,
    half-warp): a 64-bit LDS is served per half-warp, so 16 distinct 8-byte
    bank pairs per half-warp is conflict-free."""

    def __init__(self, e_col, e_cls, e_q, e_lane, counts, col_at_pos, pos_of_col, n_steps, n_cls, ubase_dbl,
                 out_of_col):
        self.e_col, self.e_cls, self.e_q, self.e_lane = e_col, e_cls, e_q, e_lane
        self.col_at_pos, self.pos_of_col = col_at_pos.copy(), pos_of_col.copy()
        self.n_cls, self.ubase = n_cls, ubase_dbl
        self.sw = (5 * np.arange(n_steps)) & 15
        n_pos = len(col_at_pos)
        self.n_cells = (n_pos // 32) * n_cls * 2
        cp = counts[np.maximum(col_at_pos, 0)] * (col_at_pos >= 0)[:, None]
        self.R = np.repeat(cp.reshape(-1, 32, n_cls).max(1).reshape(-1), 2)  # rows per cell
        self.by_q = [np.nonzero(e_q == q)[0] for q in range(n_steps)]
        self.by_col = {}
        for i, cc in enumerate(e_col.tolist()):
            self.by_col.setdefault(cc, []).append(i)
        key = {}
        for cc in range(len(pos_of_col)):
            key.setdefault((int(out_of_col[cc]), counts[cc].tobytes()), []).append(cc)
        self.twins = [v for v in key.values() if len(v) > 1]
        self.H = np.zeros((self.n_cells, 16), np.int64)
        self._apply(np.arange(len(e_col)), 1)

    def cells(self, idx):
        pos = self.pos_of_col[self.e_col[idx]]
        return ((pos >> 5) * self.n_cls + self.e_cls[idx]) * 2 + ((pos >> 4) & 1)

    def banks(self, idx):
        return (self.ubase + (self.e_lane[idx] ^ self.sw[self.e_q[idx]])) & 15

    def cost_cells(self, cells):
        # U wavefronts of a half-warp over the chunk's rows >= max(rows, max
        # bank-pair load); _assign_rows gets close to it
        cells = np.unique(cells)
        return int(np.maximum(self.R[cells], self.H[cells].max(1)).sum())

    def total(self):
        return self.cost_cells(np.arange(self.n_cells))

    def _apply(self, idx, sign):
        np.add.at(self.H, (self.cells(idx), self.banks(idx)), sign)

    def _swap(self, p1, p2):
        c1, c2 = int(self.col_at_pos[p1]), int(self.col_at_pos[p2])
        self.col_at_pos[p1], self.col_at_pos[p2] = c2, c1
        if c1 >= 0:
            self.pos_of_col[c1] = p2
        if c2 >= 0:
            self.pos_of_col[c2] = p1

    def run(self, moves, seed=12345):
        rng = np.random.default_rng(seed)
        n_steps = len(self.sw)
        for _ in range(moves):
            if rng.random() < 0.5 and n_steps:
                q = int(rng.integers(n_steps))
                idx = self.by_q[q]
                if not len(idx):
                    continue
                cells = np.unique(self.cells(idx))
                before = self.cost_cells(cells)
                old = self.sw[q]
                self._apply(idx, -1)
                self.sw[q] = int(rng.integers(16))
                self._apply(idx, 1)
                if self.cost_cells(cells) > before:
                    self._apply(idx, -1)
                    self.sw[q] = old
                    self._apply(idx, 1)
                continue
            # swap two positions inside one chunk, or two columns of one output
            # with identical per-class counts (rows per cell stay unchanged)
            if rng.random() < 0.5 or not self.twins:
                p1 = int(rng.integers(len(self.col_at_pos)))
                p2 = (p1 & ~31) + int(rng.integers(32))
            else:
                tw = self.twins[int(rng.integers(len(self.twins)))]
                i1, i2 = rng.choice(len(tw), 2, replace=False)
                p1, p2 = int(self.pos_of_col[tw[int(i1)]]), int(self.pos_of_col[tw[int(i2)]])
            c1, c2 = int(self.col_at_pos[p1]), int(self.col_at_pos[p2])
            if p1 == p2 or (c1 < 0 and c2 < 0):
                continue
            idx = np.array(self.by_col.get(c1, []) + self.by_col.get(c2, []), dtype=np.int64)
            if not len(idx):
                self._swap(p1, p2)
                continue
            cells0 = self.cells(idx)
            self._swap(p1, p2)
            cells = np.unique(np.concatenate([cells0, self.cells(idx)]))
            self._swap(p1, p2)
            before = self.cost_cells(cells)
            self._apply(idx, -1)
            self._swap(p1, p2)
            self._apply(idx, 1)
            if self.cost_cells(cells) > before:
                self._apply(idx, -1)
                self._swap(p1, p2)
                self._apply(idx, 1)


def _assign_rows(lists, zero_of_bank):
    """Order each lane's gather entries over the chunk's rows (rows = the
    longest lane list) so that each row's 64-bit U loads hit as few repeated
    bank pairs per half-warp as possible: per row and half-warp a maximum
    bipartite matching lanes -> bank pairs (lanes that must take an entry this
    row first), the rest on the least-loaded bank pair.  lists[lane] =
    [(payload, bank)]; returns (rows, 32) payloads, idle lanes reading a zero
    slot on a free bank pair (zero_of_bank[bank] = payload)."""
    n_rows = max((len(x) for x in lists), default=0)
    out = np.zeros((n_rows, 32), np.int64)
    rem = [list(x) for x in lists]
    for r in range(n_rows):
        left = n_rows - r
        for half in (0, 16):
            lanes = range(half, half + 16)
            must = [ln for ln in lanes if len(rem[ln]) >= left]
            opt = sorted((ln for ln in lanes if 0 < len(rem[ln]) < left), key=lambda ln: -len(rem[ln]))
            owner, choice = {}, {}

            def augment(ln, seen):
                for item in rem[ln]:
                    bk = item[1]
                    if bk in seen:
                        continue
                    seen.add(bk)
                    if bk not in owner or augment(owner[bk], seen):
                        owner[bk] = ln
                        choice[ln] = item
                        return True
                return False

            for ln in must + opt:
                augment(ln, set())
            load = [0] * 16
            for ln, item in choice.items():
                load[item[1]] += 1
            for ln in must:
                if ln not in choice:  # forced conflict: least-loaded bank pair
                    item = min(rem[ln], key=lambda it: load[it[1]])
                    choice[ln] = item
                    load[item[1]] += 1
            free = iter(b for b in range(16) if load[b] == 0)
            for ln in lanes:
                if ln in choice:
                    rem[ln].remove(choice[ln])
                    out[r, ln] = choice[ln][0]
                else:
                    out[r, ln] = zero_of_bank[next(free, ln & 15)]
    return out


def compile_program9(couplings: list[Coupling], out_widths, *, n_inputs: int | None = None,
                     n_slices_hint: int | None = None, search: bool = True) -> HostProgram9 | None:
    """Schedule for stencil9_kernel, or None when the gather does not fit its
    encodings (> 2048 distinct coefficients) or shared memory."""
    out_widths = tuple(int(w) for w in out_widths)
    couplings = [c for c in couplings if c is not None and len(c.rows)]
    out_off = np.concatenate([[0], np.cumsum(out_widths)]).astype(np.int64)
    n_out_cols = int(out_off[-1])
    if couplings:
        s_arr = np.concatenate([np.full(len(c.rows), c.s, np.int64) for c in couplings])
        t_arr = np.concatenate([np.full(len(c.rows), c.t, np.int64) for c in couplings])
        l_arr = np.concatenate([np.asarray(c.rows, np.int64) for c in couplings])
        o_arr = np.concatenate([np.full(len(c.rows), c.o, np.int64) for c in couplings])
        k_arr = np.concatenate([np.asarray(c.cols, np.int64) for c in couplings])
        v_arr = np.concatenate([np.asarray(c.vals, np.float64) for c in couplings])
    else:
        s_arr = t_arr = l_arr = o_arr = k_arr = np.zeros(0, np.int64)
        v_arr = np.zeros(0)
    coef_tab, coef_idx = np.unique(v_arr, return_inverse=True)
    coef_idx = np.asarray(coef_idx, np.int64).reshape(-1)
    if len(coef_tab) == 0:
        coef_tab = np.zeros(1)
    if len(coef_tab) * 8 > (1 << 14):
        return None
    # groups of 128 consecutive columns per input (the last one shifted left so
    # it stays 128 wide when the input spans >= 128 columns: a column covered
    # twice is computed twice, its product slot is taken from the first group).
    # Product (s, l, t) lives at slot base + (lane0 ^ sw[q]), base = group base
    # + 128 qq + 32 c: a per-step XOR swizzle (< 16) keeps the producer's STS
    # conflict-free and spreads the gather over bank pairs.
    specs = []  # (s, col0, ncols, [(t, [l...]) ...])
    for s in np.unique(s_arr):
        sel = s_arr == s
        cols = np.unique(l_arr[sel])
        ts_s, ls_s = t_arr[sel], l_arr[sel]
        span_hi = int(cols[-1]) + 1
        i = 0
        while i < len(cols):
            col0 = int(cols[i])
            j = int(np.searchsorted(cols, col0 + GROUP_COLS))
            if span_hi >= GROUP_COLS:
                col0 = min(col0, span_hi - GROUP_COLS)
                ncols = GROUP_COLS
            else:
                ncols = span_hi - col0
            in_g = (ls_s >= col0) & (ls_s < col0 + ncols)
            gt, gl = ts_s[in_g], ls_s[in_g] - col0
            specs.append((int(s), col0, ncols, [(int(t), np.unique(gl[gt == t])) for t in np.unique(gt)]))
            i = j
    # group position g is run by warp g % warps when there are more groups
    # than warps (8): place them longest-first on the least-loaded warp that
    # still has a position, so the products phase ends together
    n_warps_prod = 16 if (S9_BIG and len(specs) <= 16) else 8
    if len(specs) > n_warps_prod:
        cap = [len(range(w, len(specs), n_warps_prod)) for w in range(n_warps_prod)]
        load = [0] * n_warps_prod
        used = [0] * n_warps_prod
        pos = [0] * len(specs)
        for gi in sorted(range(len(specs)), key=lambda g: (-len(specs[g][3]), g)):
            w = min((w for w in range(n_warps_prod) if used[w] < cap[w]), key=lambda w: (load[w], w))
            pos[gi] = w + used[w] * n_warps_prod
            used[w] += 1
            load[w] += len(specs[gi][3])
        specs = [specs[g] for g in np.argsort(pos)]
    group_info = []
    step_rec = []
    prod_of = {}  # (s, l, t) -> (q, base, lane0)
    n_ubuf = 0
    executed = 0
    for s, col0, ncols, terms in specs:
        q0 = len(step_rec)
        group_info.append((s, col0, ncols, q0))
        for qq, (t, ls) in enumerate(terms):
            step_rec.append(t)
            for l in ls:
                key = (s, col0 + int(l), t)
                if key not in prod_of:
                    prod_of[key] = (q0 + qq, n_ubuf + qq * GROUP_COLS + (int(l) // 32) * 32, int(l) % 32)
            executed += GROUP_COLS
        n_ubuf += GROUP_COLS * (len(step_rec) - q0)
    n_steps = len(step_rec)
    if n_steps and max(step_rec) >= (1 << 16):
        return None
    group_info.append((0, 0, 0, n_steps))
    zero = n_ubuf + 32  # 32 zero slots after 32 spare slots
    n_slices = n_slices_hint if n_slices_hint is not None else (int(t_arr.max()) + 1 if len(t_arr) else 1)
    ubuf_base = _ubuf_base(len(coef_tab), n_slices)
    if (ubuf_base + 8 * (n_ubuf + 64)) >= (1 << 18):
        return None
    ubase_dbl = ubuf_base // 8
    n_ent = len(v_arr)
    prod = np.array([prod_of[(int(a), int(b), int(c))] for a, b, c in zip(s_arr, l_arr, t_arr)],
                    dtype=np.int64).reshape(-1, 3)
    e_q, e_base, e_lane = prod[:, 0], prod[:, 1], prod[:, 2]
    c_arr = out_off[o_arr] + k_arr if n_ent else np.zeros(0, np.int64)
    o_of_c = np.repeat(np.arange(len(out_widths)), out_widths)
    k_of_c = np.concatenate([np.arange(w) for w in out_widths]) if n_out_cols else np.zeros(0, np.int64)
    stats_extra = {}
    sw = (5 * np.arange(n_steps)) & 15
    counts = np.zeros((n_out_cols, 1), np.int64)
    if n_ent:
        np.add.at(counts, (c_arr, 0), 1)
    col_at_pos, pos_of_col = _class_layout(counts, out_off, 1)
    zeros_e = np.zeros(n_ent, np.int64)
    if n_ent:
        bs = _BankSearch(c_arr, zeros_e, e_q, e_lane, counts, col_at_pos, pos_of_col, n_steps, 1, ubase_dbl, o_of_c)
        stats_extra["bank_model_start"] = bs.total()
        if search and SEARCH_MOVES:
            bs.run(min(SEARCH_MOVES, 8 * n_ent))
        stats_extra["bank_model"] = bs.total()
        sw, col_at_pos, pos_of_col = bs.sw, bs.col_at_pos, bs.pos_of_col
    n_chunks = len(col_at_pos) // 32
    slot = e_base + (e_lane ^ sw[e_q]) if n_ent else np.zeros(0, np.int64)
    bank = (ubase_dbl + slot) & 15
    payload = ((ubuf_base + 8 * slot) << 14) | (8 * coef_idx)
    zero_of_bank = {(ubase_dbl + zero + z) & 15: (ubuf_base + 8 * (zero + z)) << 14 for z in range(16)}
    per = {}
    pos_e = pos_of_col[c_arr] if n_ent else np.zeros(0, np.int64)
    for i in range(n_ent):
        pos = int(pos_e[i])
        per.setdefault(pos >> 5, {}).setdefault(pos & 31, []).append((int(payload[i]), int(bank[i])))
    blocks = []
    zero_word = zero_of_bank[min(zero_of_bank)]
    for ch in range(n_chunks):
        lanes = per.get(ch)
        rows = _assign_rows([lanes.get(ln, []) for ln in range(32)], zero_of_bank) if lanes else \
            np.zeros((0, 32), np.int64)
        if len(rows) % 2:  # even row count: the kernel reads rows in pairs
            rows = np.vstack([rows, np.full((1, 32), zero_word, np.int64)])
        blocks.append(rows.astype(np.uint32))
    # chunk slot j is gathered by warp j % warps (the launcher's warp count):
    # balance the warps' total gather rows (longest-processing-time first),
    # since the barrier after the gather waits for the busiest warp
    n_groups = len(group_info) - 1
    warps = stencil9_warps(n_groups, n_chunks)
    per_warp = -(-n_chunks // warps) if n_chunks else 0
    n_slots = per_warp * warps
    order = sorted(range(n_chunks), key=lambda c: (-len(blocks[c]), c))
    slot_of_chunk = {}
    load = [0] * warps
    used = [0] * warps
    for c in order:
        w = min((w for w in range(warps) if used[w] < per_warp), key=lambda w: (load[w], w))
        slot_of_chunk[c] = w + used[w] * warps
        used[w] += 1
        load[w] += len(blocks[c])
    stats_extra["gather_rows_max_warp"] = int(max(load)) if load else 0
    chunk_meta = [(0, 0)] * n_slots
    out_col = -np.ones(n_slots * 32, np.int64)
    ents, off = [], 0
    inv = {v: c for c, v in slot_of_chunk.items()}
    for j in range(n_slots):
        c = inv.get(j)
        if c is None:
            chunk_meta[j] = (0, off)
            continue
        blk = blocks[c]
        chunk_meta[j] = (len(blk), off)
        # row pairs interleaved per lane: word 2*(32*e + lane) + {0, 1} holds
        # rows 2e and 2e+1 of the lane (one 8-byte load per pair)
        ents.append(blk.reshape(-1, 2, 32).transpose(0, 2, 1).reshape(-1))
        off += blk.size
        cols = col_at_pos[32 * c: 32 * c + 32]
        safe = np.maximum(cols, 0)
        out_col[32 * j: 32 * j + 32] = np.where(cols >= 0, (o_of_c[safe] << 24) | k_of_c[safe], -1)
    stats_extra["gather_rows"] = int(sum(len(b) for b in blocks))
    stats_extra["warps"] = warps
    gather_ptr = np.array(chunk_meta, dtype=np.int64).reshape(-1) if chunk_meta else np.zeros(2, np.int64)
    ent = np.concatenate(ents).astype(np.uint32) if ents else np.zeros(0, np.uint32)
    n_gather = int(len(ent))
    useful = len(prod_of)
    step_words = (np.array(step_rec, dtype=np.int64) | (np.asarray(sw, np.int64) << 16)) if n_steps else np.zeros(1)
    stats = {"mode": "stencil9", "n_products": int(useful),
             "n_groups": len(group_info) - 1, "n_steps": n_steps,
             "lane_efficiency": float(useful / executed) if executed else 1.0,
             "n_gather": int(n_ent), "n_gather_words": n_gather, "n_ubuf": int(n_ubuf),
             "n_coef": int(len(coef_tab)), **stats_extra}
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
    return HostProgram9(
        n_groups=len(group_info) - 1,
        n_steps=n_steps,
        n_ubuf=int(n_ubuf),
        n_out_cols=n_out_cols,
        n_coef=int(len(coef_tab)),
        n_gather=n_gather,
        group_info=i32(np.array(group_info, dtype=np.int64).reshape(-1)),
        step_rec=i32(step_words),
        coef_tab=np.ascontiguousarray(coef_tab if len(coef_tab) else np.zeros(1)),
        gather_ptr=i32(gather_ptr),
        gather_ent=np.ascontiguousarray(ent if n_gather else np.zeros(1, np.uint32)),
        out_col=i32(out_col if len(out_col) else -np.ones(1)),
        out_widths=out_widths,
        stats=stats,
        n_slices=n_slices,
        warps=warps,
    )


def emulate9(prog: HostProgram9, mats, inputs, inits, alpha, beta):
    """NumPy emulation of stencil9_kernel's schedule (test helper): mats[t]
    is slice t as a SciPy matrix, inputs[s] the (n, width) input arrays."""
    n_rows = mats[0].shape[0]
    ub = np.zeros((n_rows, prog.n_ubuf + 64))
    ubase = _ubuf_base(prog.n_coef, prog.n_slices)
    gi = prog.group_info.reshape(-1, 4)
    base = 0
    for g in range(prog.n_groups):
        s, col0, ncols, q0 = (int(v) for v in gi[g])
        q1 = int(gi[g + 1, 3])
        x = inputs[s]
        for q in range(q0, q1):
            t, sw = int(prog.step_rec[q]) & 0xFFFF, int(prog.step_rec[q]) >> 16
            for c in range(GROUP_COLS // 32):
                for lane in range(32):
                    col = col0 + min(32 * c + lane, ncols - 1)
                    ub[:, base + (q - q0) * GROUP_COLS + c * 32 + (lane ^ sw)] = mats[t] @ x[:, col]
        base += GROUP_COLS * (q1 - q0)
    n_chunks = (len(prog.out_col) // 32) if prog.n_out_cols else 0
    meta = prog.gather_ptr.reshape(-1, 2)
    acc = np.zeros((n_rows, n_chunks * 32))
    for ch in range(n_chunks):
        cnt, off = int(meta[ch, 0]), int(meta[ch, 1])
        for e in range(cnt):
            for lane in range(32):
                w = int(prog.gather_ent[off + 2 * (32 * (e // 2) + lane) + e % 2])
                acc[:, ch * 32 + lane] += prog.coef_tab[(w & 0x3FFF) // 8] * ub[:, ((w >> 14) - ubase) // 8]
    outs = [np.zeros((n_rows, w)) for w in prog.out_widths]
    for pos in range(n_chunks * 32):
        oc = int(prog.out_col[pos])
        if oc < 0:
            continue
        o, k = oc >> 24, oc & 0xFFFFFF
        y = alpha[o] * acc[:, pos]
        if inits[o] is not None:
            y = y + beta[o] * inits[o][:, k]
        outs[o][:, k] = y
    return outs
