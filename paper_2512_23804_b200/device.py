"""Device-side objects: the shared CSR pattern with t-stacked values, compiled
coupling programs, and the thin wrappers that launch them through the C ABI.

PyTorch is used only to own device buffers and to provide the stream.
"""

from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from .program import HostProgram, HostProgram9, compile_program, compile_program9

__all__ = [
    "DevicePattern",
    "DeviceProgram",
    "as_device_state",
    "device",
    "run_program",
]

F64 = torch.float64
# set SGKKT_FAST9=0 to force the general program kernel (A/B testing)
import os as _os

FAST9 = _os.environ.get("SGKKT_FAST9", "1") != "0"
# Product-heavy single-input programs on a Q1 grid pattern (the config-4
# matvec) run the grid-form kernel: sliding V window along grid-line segments
# (3 new neighbour rows per mesh row instead of 9), bit-identical.  With the
# round-1 named-barrier hand-over it measured 1.141 ms against 1.092 ms for
# the pattern-indexed kernel; on the TMA/mbarrier pipeline 1.043 ms against
# 1.070 ms (gpurun_out/g56_ab.log) — on by default, SGKKT_GRID9=0 for A/B
GRID9 = _os.environ.get("SGKKT_GRID9", "1") == "1"
# output columns one launch can hold (16 gather chunks x 256 threads in both
# kernels); wider programs are launched per column block
MAX_LAUNCH_COLS = 16 * 256


def device() -> torch.device:
    _lib.lib()  # raises when the library or a CUDA device is missing
    return torch.device("cuda", torch.cuda.current_device())


def _i32(a) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).to(device())


def _f64(a) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(device())


def as_device_state(x, shape=None) -> tuple[torch.Tensor, bool]:
    """(tensor on the device, came_from_numpy).  NumPy inputs (any memory
    order) are copied to a node-major float64 CUDA tensor."""
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            x = x.to(device(), non_blocking=x.is_pinned())
            host = True
        else:
            host = False
        if x.dtype != F64:
            raise ValueError(f"expected float64 data, got {x.dtype}")
        if shape is not None and tuple(x.shape) != tuple(shape):
            raise ValueError(f"state shape {tuple(x.shape)} does not match {tuple(shape)}")
        return x if x.is_contiguous() else x.contiguous(), host
    arr = np.asarray(x, dtype=np.float64)
    if shape is not None and arr.shape != tuple(shape):
        raise ValueError(f"state shape {arr.shape} does not match {tuple(shape)}")
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.to(device(), non_blocking=t.is_pinned()), True


class DevicePattern:
    """One CSR pattern shared by a list of sparse matrices (the union of
    their structures) with the values of all of them stacked per row:
    vals[rowptr[i]*T + t*len_i + jj].  Structural entries of one matrix that
    are absent from another are stored as exact zeros there."""

    def __init__(self, mats: list[sp.spmatrix]):
        if not mats:
            raise ValueError("need at least one matrix")
        n, m = mats[0].shape
        for a in mats:
            if a.shape != (n, m):
                raise ValueError("operator matrices must share their size")
        csrs = [sp.csr_matrix(a) for a in mats]
        for a in csrs:
            a.sum_duplicates()
            a.sort_indices()
        if all(a.nnz == csrs[0].nnz and np.array_equal(a.indptr, csrs[0].indptr)
               and np.array_equal(a.indices, csrs[0].indices) for a in csrs):
            indptr, indices = csrs[0].indptr.astype(np.int64), csrs[0].indices.astype(np.int64)
            std = np.stack([a.data for a in csrs]) if csrs[0].nnz else np.zeros((len(csrs), 0))
        else:
            rows = np.concatenate([np.repeat(np.arange(n), np.diff(a.indptr)) for a in csrs])
            cols = np.concatenate([a.indices for a in csrs]).astype(np.int64)
            keys = np.unique(rows.astype(np.int64) * m + cols)
            r_u, c_u = np.divmod(keys, m)
            indptr = np.concatenate([[0], np.cumsum(np.bincount(r_u, minlength=n))]).astype(np.int64)
            indices = c_u
            std = np.zeros((len(csrs), len(keys)))
            for t, a in enumerate(csrs):
                ar = np.repeat(np.arange(n), np.diff(a.indptr)).astype(np.int64)
                pos = np.searchsorted(keys, ar * m + a.indices.astype(np.int64))
                std[t, pos] = a.data
        self.n_rows = n
        self.n_cols = m
        self.n_slices = len(csrs)
        self.nnz = int(len(indices))
        self.indptr = indptr
        self.indices = indices
        self.slice_data = std  # (T, nnz) in CSR order, host copy for checks
        lens = np.diff(indptr)
        self.max_row_nnz = int(lens.max()) if n else 0
        # row-block, slice-major device layout
        row_of = np.repeat(np.arange(n), lens)
        jj = np.arange(self.nnz) - indptr[row_of]
        dst = (indptr[row_of] * self.n_slices)[None, :] + np.arange(self.n_slices)[:, None] * lens[row_of][None, :] + jj[None, :]
        vals = np.empty(self.nnz * self.n_slices)
        vals[dst.ravel()] = std.ravel()
        self._rowptr = _i32(indptr)
        self._colind = _i32(indices)
        self._vals = _f64(vals)
        self.struct = _lib.Pattern(
            n_rows=n,
            n_slices=self.n_slices,
            max_row_nnz=self.max_row_nnz,
            pad=0,
            rowptr=self._rowptr.data_ptr(),
            colind=self._colind.data_ptr(),
            vals=self._vals.data_ptr(),
        )

    @classmethod
    def assemble_q1(cls, grid, fields, with_mass: bool = True) -> "DevicePattern":
        """Device-assembled pattern: slices = the Q1
        stiffness matrices of the coefficient fields (+ the mass matrix as
        the last slice), built by csrc/assemble.cu directly into both device
        layouts.  `fields` is a (T, n_elements, 4) float64 array or CUDA
        tensor of Gauss-point samples (reference fem.py:171-206)."""
        from . import fem

        f = fields if isinstance(fields, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(fields, np.float64))
        f = f.to(device(), dtype=F64).contiguous()
        if f.dim() != 3 or f.shape[1] != grid.n_elements or f.shape[2] != 4:
            raise ValueError("fields must have shape (T, n_elements, 4)")
        T = int(f.shape[0])
        S = T + (1 if with_mass else 0)
        if S == 0:
            raise ValueError("nothing to assemble")
        struct_m = fem.assemble_mass(grid)  # the shared 9-point structure
        self = cls.__new__(cls)
        n = struct_m.shape[0]
        self.n_rows = self.n_cols = n
        self.n_slices = S
        self.nnz = int(struct_m.nnz)
        self.indptr = struct_m.indptr.astype(np.int64)
        self.indices = struct_m.indices.astype(np.int64)
        self._slice_data = None
        lens = np.diff(self.indptr)
        self.max_row_nnz = int(lens.max()) if n else 0
        self._rowptr = _i32(self.indptr)
        self._colind = _i32(self.indices)
        self._vals = torch.empty(max(self.nnz * S, 1), dtype=F64, device=device())
        self._colind9 = torch.empty((n, 9), dtype=torch.int32, device=device())
        self._coef10 = torch.empty((n, S, 10), dtype=F64, device=device())
        stiff_q = np.ascontiguousarray(fem._STIFF_Q, np.float64)
        mass_ref = np.ascontiguousarray(fem._MASS_REF, np.float64)
        rc = _lib.lib().sgk_q1_assemble(
            grid.n_cells, T, f.data_ptr() if T else None, stiff_q.ctypes.data, int(with_mass),
            float(grid.quad_weight), mass_ref.ctypes.data, self._rowptr.data_ptr(), self._vals.data_ptr(),
            self._coef10.data_ptr(), self._colind9.data_ptr(), _lib.stream_ptr())
        _lib.check(rc, "sgk_q1_assemble")
        self.struct = _lib.Pattern(n_rows=n, n_slices=S, max_row_nnz=self.max_row_nnz, pad=0,
                                   rowptr=self._rowptr.data_ptr(), colind=self._colind.data_ptr(),
                                   vals=self._vals.data_ptr())
        self._p9 = _lib.Pattern9(n_rows=n, n_slices=S, colind9=self._colind9.data_ptr(),
                                 coef10=self._coef10.data_ptr())
        return self

    @property
    def slice_data(self) -> np.ndarray:
        """(T, nnz) slice values in CSR order (host copy; fetched from the
        device for device-assembled patterns)."""
        if self._slice_data is None:
            lens = np.diff(self.indptr)
            row_of = np.repeat(np.arange(self.n_rows), lens)
            jj = np.arange(self.nnz) - self.indptr[row_of]
            src = (self.indptr[row_of] * self.n_slices)[None, :] + np.arange(self.n_slices)[:, None] * lens[row_of][None, :] + jj[None, :]
            self._slice_data = self._vals.cpu().numpy()[src]
        return self._slice_data

    @slice_data.setter
    def slice_data(self, v):
        self._slice_data = v

    def pattern9(self):
        """Padded 9-entry layout for the fast path (None if a row is longer)."""
        if self.max_row_nnz > 9:
            return None
        if getattr(self, "_p9", None) is None:
            n, T = self.n_rows, self.n_slices
            lens = np.diff(self.indptr)
            row_of = np.repeat(np.arange(n), lens)
            jj = np.arange(self.nnz) - self.indptr[row_of]
            cols9 = np.zeros((n, 9), dtype=np.int64)
            last = np.where(lens > 0, self.indices[np.maximum(self.indptr[1:] - 1, 0)], 0) if self.nnz else np.zeros(n, np.int64)
            cols9[:] = last[:, None]
            cols9[row_of, jj] = self.indices
            coef = np.zeros((n, T, 10))
            for t in range(T):
                coef[row_of, t, jj] = self.slice_data[t]
            self._colind9 = _i32(cols9)
            self._coef10 = _f64(coef)
            self._p9 = _lib.Pattern9(n_rows=n, n_slices=T, colind9=self._colind9.data_ptr(),
                                     coef10=self._coef10.data_ptr())
        return self._p9

    def grid9(self):
        """(nx, ny, coefg) when the pattern is the Q1 9-point stencil of an
        nx x ny grid in natural node order (neighbours of p = iy*nx + ix are
        p + dy*nx + dx, every in-grid neighbour present), else None.  coefg =
        the t-stacked values in stencil-position order (sgk_grid9 layout)."""
        if not hasattr(self, "_grid9"):
            self._grid9 = None
            n = self.n_rows
            if self.max_row_nnz <= 9 and n >= 9 and self.n_cols == n and self.pattern9() is not None:
                row0 = self.indices[self.indptr[0]:self.indptr[1]]
                nx = int(row0[2]) if len(row0) == 4 else 0
                if nx >= 3 and n % nx == 0:
                    ny = n // nx
                    p = np.arange(n, dtype=np.int64)
                    iy, ix = p // nx, p % nx
                    want = []
                    for dy in (-1, 0, 1):
                        for dx in (-1, 0, 1):
                            ok = (iy + dy >= 0) & (iy + dy < ny) & (ix + dx >= 0) & (ix + dx < nx)
                            want.append(np.where(ok, p + dy * nx + dx, -1))
                    want = np.stack(want, 1)
                    cnt = (want >= 0).sum(1)
                    if np.array_equal(cnt, np.diff(self.indptr)):
                        cols = np.sort(np.where(want >= 0, want, n + 1), 1)[:, :9]
                        row_of = np.repeat(p, cnt)
                        jj = np.arange(self.nnz) - self.indptr[row_of]
                        if np.array_equal(cols[row_of, jj], self.indices):
                            p9 = self.pattern9()
                            coefg = torch.empty((n, self.n_slices, 10), dtype=F64, device=device())
                            rc = _lib.lib().sgk_grid9_coef(n, self.n_slices, nx, p9.colind9, p9.coef10,
                                                           coefg.data_ptr(), _lib.stream_ptr())
                            _lib.check(rc, "sgk_grid9_coef")
                            self._grid9 = (nx, ny, coefg)
        return self._grid9

    @property
    def algorithmic_bytes(self) -> int:
        """t-stacked values (8 B) + int32 pattern, read once."""
        return 8 * self.n_slices * self.nnz + 4 * (self.nnz + self.n_rows + 1)


class _GenericProgram:
    def __init__(self, host: HostProgram):
        self.host = host
        self._bufs = [
            _i32(host.lane_item if host.lane_item.size else [0]),
            _i32(host.group_step0),
            _i32(host.step_term if host.step_term.size else [0]),
            _i32(host.phase_group0),
            _i32(host.gather_ptr),
            _i32(host.gather_slot if host.gather_slot.size else [0]),
            _f64(host.gather_coef if host.gather_coef.size else [0.0]),
            _i32(host.out_col if host.out_col.size else [0]),
        ]
        # compact gather: one 32-bit word per entry (slot | coefficient index
        # << 16) when the distinct coefficients fit a small shared table
        # (config 3: 12.8 k entries, 16 distinct values: 51 KB instead of 154 KB
        # of table read per mesh row)
        n_coef = 0
        if host.gather_coef.size:
            tab, idx = np.unique(host.gather_coef, return_inverse=True)
            if len(tab) <= 2048 and host.max_phase_slots <= 65536:
                n_coef = len(tab)
                words = (np.asarray(host.gather_slot, np.int64) | (np.asarray(idx, np.int64).reshape(-1) << 16))
                self._bufs += [torch.as_tensor(words.astype(np.uint32).view(np.int32)).to(device()), _f64(tab)]
        b = self._bufs
        self.struct = _lib.Program(
            n_groups=host.n_groups, n_phases=host.n_phases, n_out_cols=host.n_out_cols,
            max_phase_slots=host.max_phase_slots, lane_item=b[0].data_ptr(), group_step0=b[1].data_ptr(),
            step_term=b[2].data_ptr(), phase_group0=b[3].data_ptr(), gather_ptr=b[4].data_ptr(),
            gather_slot=b[5].data_ptr(), gather_coef=b[6].data_ptr(), out_col=b[7].data_ptr(),
            n_coef=n_coef, pad=0, gather_word=b[8].data_ptr() if n_coef else None,
            coef_tab=b[9].data_ptr() if n_coef else None,
        )


class _Program9:
    def __init__(self, host: HostProgram9):
        self.host = host
        self._bufs = [
            _i32(host.group_info), _i32(host.step_rec), _f64(host.coef_tab), _i32(host.gather_ptr),
            torch.as_tensor(host.gather_ent.view(np.int32)).to(device()), _i32(host.out_col),
        ]
        b = self._bufs
        self.struct = _lib.Program9(
            n_groups=host.n_groups, n_steps=host.n_steps, n_ubuf=host.n_ubuf, n_out_cols=host.n_out_cols,
            n_coef=host.n_coef, n_gather=host.n_gather, n_slices=host.n_slices,
            n_chunks=len(host.out_col) // 32 if host.n_out_cols else 0,
            group_info=b[0].data_ptr(), step_rec=b[1].data_ptr(),
            coef_tab=b[2].data_ptr(), gather_ptr=b[3].data_ptr(), gather_ent=b[4].data_ptr(),
            out_col=b[5].data_ptr(),
            coef8=(ctypes.c_double * 8)(*[float(v) for v in np.asarray(host.coef_tab, np.float64).reshape(-1)[:8]]),
        )


class DeviceProgram:
    """A compiled coupling program.  Two device schedules are derived from the
    same couplings on demand: the 9-point fast path (stencil9_kernel) and the
    general one (program_kernel)."""

    def __init__(self, couplings, out_widths, n_inputs: int | None = None):
        self.couplings = [c for c in couplings if c is not None]
        self._widths = tuple(int(w) for w in out_widths)
        self.n_inputs = n_inputs
        self._generic = None
        self._fast9 = {}

    @property
    def out_widths(self) -> tuple[int, ...]:
        return self._widths

    @property
    def generic(self) -> _GenericProgram:
        if self._generic is None:
            self._generic = _GenericProgram(compile_program(self.couplings, self._widths, n_inputs=self.n_inputs))
        return self._generic

    def fast9(self, n_slices: int) -> _Program9 | None:
        """9-point schedule for a pattern with `n_slices` value slices (the
        gather entries encode shared-memory offsets that depend on it)."""
        if n_slices not in self._fast9:
            host = compile_program9(self.couplings, self._widths, n_inputs=self.n_inputs, n_slices_hint=n_slices)
            self._fast9[n_slices] = _Program9(host) if host is not None else None
        return self._fast9[n_slices]

    def column_parts(self, max_cols: int):
        """Single-output sub-programs covering <= max_cols output columns each
        (one CTA holds at most MAX_LAUNCH_COLS output columns of a row): a list
        of (output index, first column, sub-program)."""
        key = ("parts", max_cols)
        parts = self._fast9.get(key)
        if parts is None:
            from .program import Coupling

            parts = []
            for o, w in enumerate(self._widths):
                for k0 in range(0, w, max_cols):
                    k1 = min(w, k0 + max_cols)
                    sub = []
                    for c in self.couplings:
                        if c.o != o:
                            continue
                        keep = (c.cols >= k0) & (c.cols < k1)
                        if np.any(keep):
                            sub.append(Coupling(s=c.s, o=0, t=c.t, rows=c.rows[keep], cols=c.cols[keep] - k0,
                                                vals=c.vals[keep]))
                    parts.append((o, k0, DeviceProgram(sub, (k1 - k0,), n_inputs=self.n_inputs)))
            self._fast9[key] = parts
        return parts

    @property
    def host(self):
        """Schedule statistics of the fast path compiled last (else the general one)."""
        for k, f in self._fast9.items():
            if f is not None and not isinstance(k, tuple):
                return f.host
        return self.generic.host


def _view(t: torch.Tensor | None, col0: int = 0) -> _lib.View:
    if t is None:
        return _lib.View(ptr=None, ld=0, col0=0, pad=0)
    if t.dim() != 2 or t.stride(1) != 1 or t.dtype != F64 or not t.is_cuda:
        raise ValueError("device views must be 2-D float64 CUDA tensors with unit column stride")
    return _lib.View(ptr=t.data_ptr(), ld=t.stride(0), col0=col0, pad=0)


def _grid_seg_len(nx: int, n_rows: int) -> int:
    """Grid-line segment length for stencil9_grid_kernel's CTA walk: the
    candidate (<= 64 rows, >= 8) with the fewest row steps per CTA,
    ceil(segments / CTAs) * length, with at least one segment per CTA."""
    env = _os.environ.get("SGKKT_GRID_SEG")
    if env:
        return max(1, int(env))
    ctas = _lib.sm_count()
    best = None
    for k in range(1, 33):
        seg = -(-nx // k)
        if seg > 64:
            continue
        n_seg = -(-n_rows // nx) * k + 1
        cost = -(-n_seg // ctas) * (seg + 0.5)  # + a segment restart (full window load)
        if best is None or cost < best[0]:
            best = (cost, seg)
        if seg < 8:
            break
    return best[1] if best else max(1, nx)


def run_program(
    pattern: DevicePattern,
    program: DeviceProgram,
    inputs: list[tuple[torch.Tensor, int]],
    outputs: list[tuple[torch.Tensor, int]],
    inits: list[tuple[torch.Tensor, int] | None] | None = None,
    alpha: list[float] | None = None,
    beta: list[float] | None = None,
    threads: int = 256,
    stream: torch.cuda.Stream | None = None,
    rows: tuple[int, int] | None = None,
) -> None:
    """Launch program_kernel: outputs[o][:, col0+k] = alpha*gather + beta*init.
    `rows=(a, b)` restricts the launch to mesh rows [a, b) (9-point fast path
    only; used by the pipelined host-buffer path)."""
    n_out = len(outputs)
    if n_out != len(program.out_widths):
        raise ValueError("output count does not match the program")
    for (t, c0), w in zip(outputs, program.out_widths):
        if t.shape[0] != pattern.n_rows or c0 + w > t.shape[1]:
            raise ValueError("output view does not fit the program")
    if sum(program.out_widths) > MAX_LAUNCH_COLS:
        # wider than one CTA's output columns: one launch per column block
        inits_l = inits or [None] * n_out
        for o, k0, sub in program.column_parts(MAX_LAUNCH_COLS):
            t, c0 = outputs[o]
            ini = inits_l[o]
            run_program(pattern, sub, inputs, [(t, c0 + k0)], [(ini[0], ini[1] + k0) if ini is not None else None],
                        alpha=[(alpha or [1.0] * n_out)[o]], beta=[(beta or [1.0] * n_out)[o]], threads=threads,
                        stream=stream, rows=rows)
        return
    for t, c0 in inputs:
        if t.shape[0] != pattern.n_cols:
            raise ValueError("input rows do not match the operator")
    in_arr = (_lib.View * max(1, len(inputs)))(*[_view(t, c) for t, c in inputs])
    out_arr = (_lib.View * n_out)(*[_view(t, c) for t, c in outputs])
    inits = inits or [None] * n_out
    init_arr = (_lib.View * n_out)(*[_view(*i) if i is not None else _view(None) for i in inits])
    a = (ctypes.c_double * n_out)(*(alpha or [1.0] * n_out))
    b = (ctypes.c_double * n_out)(*(beta or [1.0] * n_out))
    lib = _lib.lib()
    p9 = pattern.pattern9() if FAST9 else None
    f9 = program.fast9(pattern.n_slices) if p9 is not None else None
    if rows is not None:
        if f9 is None:
            raise ValueError("row-range launches need the 9-point fast path")
        r0, r1 = rows
        if not 0 <= r0 <= r1 <= pattern.n_rows:
            raise ValueError("row range out of bounds")
        p9 = _lib.Pattern9(n_rows=r1 - r0, n_slices=p9.n_slices, colind9=p9.colind9 + 4 * 9 * r0,
                           coef10=p9.coef10 + 8 * 10 * p9.n_slices * r0)
        for arr in (out_arr, init_arr):
            for v in arr:
                if v.ptr:
                    v.ptr = v.ptr + 8 * v.ld * r0
    if f9 is not None and GRID9 and len(inputs) == 1 and n_out == 1:
        h9 = f9.host
        g9 = pattern.grid9()
        gi = h9.group_info.reshape(-1, 4)[:-1]
        # product-heavy single-output programs of full 128-column groups
        # (the config-4 matvec): warp-specialised grid kernel, sliding V
        if g9 is not None and 6 <= h9.n_groups <= 8 and bool(np.all(gi[:, 2] == 128)):
            nx, ny, coefg = g9
            r0, r1 = rows if rows is not None else (0, pattern.n_rows)
            gp = _lib.Grid9(n_rows=r1 - r0, n_slices=pattern.n_slices, nx=nx, ny=ny, row0=r0,
                            seg_len=_grid_seg_len(nx, r1 - r0), coefg=coefg.data_ptr())
            rc = lib.sgk_stencil9_grid_apply(ctypes.byref(gp), ctypes.byref(f9.struct), len(inputs), in_arr,
                                             n_out, out_arr, init_arr, a, b, _lib.stream_ptr(stream))
            if rc != -3:
                _lib.check(rc, "sgk_stencil9_grid_apply")
                return
    if f9 is not None:
        h9 = f9.host
        warps = h9.warps
        rc = lib.sgk_stencil9_apply(ctypes.byref(p9), ctypes.byref(f9.struct), len(inputs), in_arr,
                                    n_out, out_arr, init_arr, a, b, 32 * warps, _lib.stream_ptr(stream))
        if rc != -3:  # -3: does not fit in shared memory -> general kernel
            _lib.check(rc, "sgk_stencil9_apply")
            return
        if rows is not None:
            # the general kernel walks the full-height pattern: never combine
            # it with the row-shifted output views of a row-range launch
            raise RuntimeError("row-range launch: the 9-point program does not fit in shared memory")
    rc = lib.sgk_program_apply(
        ctypes.byref(pattern.struct), ctypes.byref(program.generic.struct), len(inputs), in_arr, n_out,
        out_arr, init_arr, a, b, threads, _lib.stream_ptr(stream),
    )
    _lib.check(rc, "sgk_program_apply")
