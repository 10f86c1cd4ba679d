"""ctypes binding of libsgkkt_b200.so (the C ABI declared in include/sgkkt_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every device entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

__all__ = [
    "lib",
    "check",
    "Pattern",
    "Program",
    "View",
    "TriFactor",
    "SegView",
    "FastDiag",
    "stream_ptr",
    "library_path",
    "launch_count",
]

_HERE = Path(__file__).resolve().parent
_LIBNAME = "libsgkkt_b200.so"

MAX_IO = 4
MAX_MDOT = 8

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p


class Pattern(ctypes.Structure):
    _fields_ = [
        ("n_rows", c_i32),
        ("n_slices", c_i32),
        ("max_row_nnz", c_i32),
        ("pad", c_i32),
        ("rowptr", c_vp),
        ("colind", c_vp),
        ("vals", c_vp),
    ]


class Program(ctypes.Structure):
    _fields_ = [
        ("n_groups", c_i32),
        ("n_phases", c_i32),
        ("n_out_cols", c_i32),
        ("max_phase_slots", c_i32),
        ("lane_item", c_vp),
        ("group_step0", c_vp),
        ("step_term", c_vp),
        ("phase_group0", c_vp),
        ("gather_ptr", c_vp),
        ("gather_slot", c_vp),
        ("gather_coef", c_vp),
        ("out_col", c_vp),
        ("n_coef", c_i32),
        ("pad", c_i32),
        ("gather_word", c_vp),
        ("coef_tab", c_vp),
    ]


class Pattern9(ctypes.Structure):
    _fields_ = [("n_rows", c_i32), ("n_slices", c_i32), ("colind9", c_vp), ("coef10", c_vp)]


class Grid9(ctypes.Structure):
    _fields_ = [("n_rows", c_i32), ("n_slices", c_i32), ("nx", c_i32), ("ny", c_i32), ("row0", c_i32),
                ("seg_len", c_i32), ("coefg", c_vp)]


class Program9(ctypes.Structure):
    _fields_ = [
        ("n_groups", c_i32), ("n_steps", c_i32), ("n_ubuf", c_i32), ("n_out_cols", c_i32),
        ("n_coef", c_i32), ("n_gather", c_i32), ("n_slices", c_i32), ("n_chunks", c_i32), ("group_info", c_vp),
        ("step_rec", c_vp),
        ("coef_tab", c_vp), ("gather_ptr", c_vp), ("gather_ent", c_vp), ("out_col", c_vp),
        ("coef8", c_dbl * 8),
    ]


class View(ctypes.Structure):
    _fields_ = [("ptr", c_vp), ("ld", c_i64), ("col0", c_i32), ("pad", c_i32)]


class TriFactor(ctypes.Structure):
    _fields_ = [
        ("n", c_i32),
        ("lower", c_i32),
        ("rowptr", c_vp),
        ("colind", c_vp),
        ("vals", c_vp),
        ("diag_inv", c_vp),
        ("order", c_vp),
        ("flags", c_vp),
        ("ticket", c_vp),
    ]


class TriGroups(ctypes.Structure):
    _fields_ = [
        ("n", c_i32), ("n_groups", c_i32), ("reversed", c_i32), ("pad", c_i32), ("rowptr", c_vp), ("split", c_vp), ("colind", c_vp), ("vals", c_vp),
        ("group_ptr", c_vp), ("group_order", c_vp), ("gdep_ptr", c_vp), ("gdep", c_vp), ("work_row", c_vp),
        ("io_row", c_vp),
        ("diag_inv", c_vp), ("flags", c_vp), ("ticket", c_vp), ("minv_ptr", c_vp), ("minv", c_vp),
        ("dense_g0", c_i32), ("dense_nb", c_i32), ("dense_r0", c_i32), ("dense_pad", c_i32), ("dense", c_vp),
    ]


class TriWide(ctypes.Structure):
    _fields_ = [
        ("n", c_i32), ("n_groups", c_i32), ("n_tiles", c_i32), ("reversed", c_i32), ("rowptr", c_vp),
        ("colind", c_vp), ("vals", c_vp), ("group_ptr", c_vp), ("tile_group", c_vp), ("tile_seg", c_vp),
        ("tile_dep_ptr", c_vp), ("tile_dep", c_vp), ("group_ntiles", c_vp), ("seg_row", c_vp), ("seg_e0", c_vp),
        ("seg_e1", c_vp), ("seg_slot", c_vp), ("row_slot_ptr", c_vp), ("row_slot", c_vp), ("work_row", c_vp),
        ("io_row", c_vp), ("minv_ptr", c_vp), ("minv", c_vp), ("flags", c_vp), ("counters", c_vp),
        ("ticket", c_vp), ("tile_kind", c_vp), ("dense_g0", c_i32), ("dense_nb", c_i32), ("dense_r0", c_i32),
        ("dense_pad", c_i32), ("dense", c_vp), ("pcol", c_vp), ("pval", c_vp), ("tile_slot", c_vp),
        ("region_inv", c_vp), ("part_rows", c_i32), ("region_pad", c_i32),
    ]


class SegView(ctypes.Structure):
    _fields_ = [("ptr", c_vp * 3), ("ld", c_i64), ("col0", c_i32), ("seg_rows", c_i32)]


class FastDiag(ctypes.Structure):
    _fields_ = [("n", c_i32), ("n_seg", c_i32), ("np", c_i32), ("pad", c_i32), ("s", c_vp), ("lam", c_vp),
                ("beta", c_dbl), ("ne", c_i32), ("hp", c_i32), ("sh", c_vp)]


_SIGNATURES = {
    "sgk_program_apply": (c_i32, [ctypes.POINTER(Pattern), ctypes.POINTER(Program), c_i32,
                                  ctypes.POINTER(View), c_i32, ctypes.POINTER(View),
                                  ctypes.POINTER(View), ctypes.POINTER(c_dbl),
                                  ctypes.POINTER(c_dbl), c_i32, c_vp]),
    "sgk_stencil9_apply": (c_i32, [ctypes.POINTER(Pattern9), ctypes.POINTER(Program9), c_i32,
                                   ctypes.POINTER(View), c_i32, ctypes.POINTER(View),
                                   ctypes.POINTER(View), ctypes.POINTER(c_dbl),
                                   ctypes.POINTER(c_dbl), c_i32, c_vp]),
    "sgk_stencil9_smem_bytes": (c_i64, [ctypes.POINTER(Pattern9), ctypes.POINTER(Program9)]),
    "sgk_stencil9_grid_apply": (c_i32, [ctypes.POINTER(Grid9), ctypes.POINTER(Program9), c_i32,
                                        ctypes.POINTER(View), c_i32, ctypes.POINTER(View),
                                        ctypes.POINTER(View), ctypes.POINTER(c_dbl),
                                        ctypes.POINTER(c_dbl), c_vp]),
    "sgk_grid9_coef": (c_i32, [c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "sgk_trisolve": (c_i32, [ctypes.POINTER(TriFactor), ctypes.POINTER(TriFactor), c_vp, c_vp,
                             ctypes.POINTER(SegView), ctypes.POINTER(SegView), c_vp, c_i32,
                             c_i32, c_vp]),
    "sgk_trisolve_chunk_cols": (c_i32, []),
    "sgk_trisolve_grouped_chunk_cols": (c_i32, []),
    "sgk_trisolve_wide_chunk_cols": (c_i32, [c_i32]),
    "sgk_trisolve_wide": (c_i32, [ctypes.POINTER(TriWide), ctypes.POINTER(TriWide), ctypes.POINTER(SegView),
                                  ctypes.POINTER(SegView), c_vp, c_vp, c_i32, c_i32, c_vp]),
    "sgk_trisolve_grouped": (c_i32, [ctypes.POINTER(TriGroups), ctypes.POINTER(TriGroups),
                                     ctypes.POINTER(SegView), ctypes.POINTER(SegView), c_vp, c_i32, c_i32,
                                     c_vp]),
    "sgk_fastdiag_work_doubles": (c_i64, [ctypes.POINTER(FastDiag), c_i32]),
    "sgk_fastdiag_solve": (c_i32, [ctypes.POINTER(FastDiag), ctypes.POINTER(SegView), ctypes.POINTER(SegView),
                                   c_vp, c_i32, c_vp]),
    "sgk_q1_assemble": (c_i32, [c_i32, c_i32, c_vp, c_vp, c_i32, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sgk_lognormal_fields": (c_i32, [c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sgk_cheb_step": (c_i32, [ctypes.POINTER(Pattern), c_i32, c_vp, c_i64, c_vp, c_vp, c_vp,
                              c_vp, c_dbl, c_vp]),
    "sgk_cheb_step_batched": (c_i32, [ctypes.POINTER(Pattern), c_i32, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp,
                                      c_vp, c_dbl, c_vp]),
    "sgk_colscale": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_i32, c_dbl, c_vp, c_vp]),
    "sgk_colscale_batched": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "sgk_reduce_blocks": (c_i32, []),
    "sgk_dot_partial": (c_i32, [c_i64, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "sgk_reduce_partials": (c_i32, [c_vp, c_i32, c_vp, c_i32, c_vp]),
    "sgk_axpby_dev": (c_i32, [c_i64, c_dbl, c_vp, c_i32, c_vp, c_dbl, c_vp, c_vp, c_vp]),
    "sgk_mgs_step": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sgk_lincomb3": (c_i32, [c_i64, c_vp, c_dbl, c_vp, c_dbl, c_vp, c_dbl, c_vp, c_vp]),
    "sgk_f2n": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp]),
    "sgk_n2f": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp]),
    "sgk_last_error": (ctypes.c_char_p, []),
    "sgk_version": (c_i32, []),
    "sgk_launch_count": (c_i64, []),
}

EXPORTED = tuple(_SIGNATURES)


def library_path() -> Path:
    return Path(os.environ.get("SGKKT_B200_LIB", str(_HERE / _LIBNAME)))


_LIB = None


def _load():
    global _LIB
    if _LIB is not None:
        return _LIB
    path = library_path()
    if not path.exists():
        raise RuntimeError(
            f"{path} is missing: build it with `make` or `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    handle = ctypes.CDLL(str(path))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = handle
    return handle


_DEVICE_OK = False


def lib():
    """The loaded library; requires a visible CUDA device (no CPU fallback).
    The device check runs until it first succeeds (a device cannot vanish
    from a running process; this is on every launch's host path)."""
    global _DEVICE_OK
    if _DEVICE_OK and _LIB is not None:
        return _LIB
    handle = _load()
    if not torch.cuda.is_available():
        raise RuntimeError("libsgkkt_b200 needs a CUDA device; none is visible (no CPU fallback)")
    _DEVICE_OK = True
    return handle


def load_without_device():
    """Load the library for symbol checks only (no compute)."""
    return _load()


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = _load().sgk_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    """cudaStream_t of `stream`, else of torch's current stream on the current
    device (the raw-pointer query skips torch.cuda.current_stream()'s Python
    wrapper: ~15 us per call, paid on every launch)."""
    if stream is not None:
        return int(stream.cuda_stream)
    if _RAW_STREAM is not None:
        return int(_RAW_STREAM(torch._C._cuda_getDevice()))
    return int(torch.cuda.current_stream().cuda_stream)


# private torch entry point (present in the torch this image ships); the
# public query above is the fallback
_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None) if hasattr(torch._C, "_cuda_getDevice") else None


def launch_count() -> int:
    return int(_load().sgk_launch_count())


_SM_COUNT = None


def sm_count() -> int:
    """SM count of the current CUDA device (cached; 148 on B200)."""
    global _SM_COUNT
    if _SM_COUNT is None:
        _SM_COUNT = int(torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count)
    return _SM_COUNT
