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
from .program import HostProgram

__all__ = [
    "DevicePattern",
    "DeviceProgram",
    "as_device_state",
    "device",
    "run_program",
]

F64 = torch.float64


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
            rowptr=self._rowptr.data_ptr(),
            colind=self._colind.data_ptr(),
            vals=self._vals.data_ptr(),
        )

    @property
    def algorithmic_bytes(self) -> int:
        """t-stacked values (8 B) + int32 pattern, read once."""
        return 8 * self.n_slices * self.nnz + 4 * (self.nnz + self.n_rows + 1)


class DeviceProgram:
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
        b = self._bufs
        self.struct = _lib.Program(
            n_groups=host.n_groups,
            n_phases=host.n_phases,
            n_out_cols=host.n_out_cols,
            max_phase_slots=host.max_phase_slots,
            lane_item=b[0].data_ptr(),
            group_step0=b[1].data_ptr(),
            step_term=b[2].data_ptr(),
            phase_group0=b[3].data_ptr(),
            gather_ptr=b[4].data_ptr(),
            gather_slot=b[5].data_ptr(),
            gather_coef=b[6].data_ptr(),
            out_col=b[7].data_ptr(),
        )

    @property
    def out_widths(self) -> tuple[int, ...]:
        return self.host.out_widths


def _view(t: torch.Tensor | None, col0: int = 0) -> _lib.View:
    if t is None:
        return _lib.View(ptr=None, ld=0, col0=0, pad=0)
    if t.dim() != 2 or t.stride(1) != 1 or t.dtype != F64 or not t.is_cuda:
        raise ValueError("device views must be 2-D float64 CUDA tensors with unit column stride")
    return _lib.View(ptr=t.data_ptr(), ld=t.stride(0), col0=col0, pad=0)


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
) -> None:
    """Launch program_kernel: outputs[o][:, col0+k] = alpha*gather + beta*init."""
    n_out = len(outputs)
    if n_out != len(program.out_widths):
        raise ValueError("output count does not match the program")
    for (t, c0), w in zip(outputs, program.out_widths):
        if t.shape[0] != pattern.n_rows or c0 + w > t.shape[1]:
            raise ValueError("output view does not fit the program")
    for t, c0 in inputs:
        if t.shape[0] != pattern.n_cols:
            raise ValueError("input rows do not match the operator")
    in_arr = (_lib.View * max(1, len(inputs)))(*[_view(t, c) for t, c in inputs])
    out_arr = (_lib.View * n_out)(*[_view(t, c) for t, c in outputs])
    inits = inits or [None] * n_out
    init_arr = (_lib.View * n_out)(*[_view(*i) if i is not None else _view(None) for i in inits])
    a = (ctypes.c_double * n_out)(*(alpha or [1.0] * n_out))
    b = (ctypes.c_double * n_out)(*(beta or [1.0] * n_out))
    rc = _lib.lib().sgk_program_apply(
        ctypes.byref(pattern.struct), ctypes.byref(program.struct), len(inputs), in_arr, n_out,
        out_arr, init_arr, a, b, threads, _lib.stream_ptr(stream),
    )
    _lib.check(rc, "sgk_program_apply")
