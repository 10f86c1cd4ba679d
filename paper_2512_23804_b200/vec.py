"""Device vector primitives over the C ABI (K6): deterministic fp64
reductions (fixed two-stage tree, no atomics) and fused updates."""

from __future__ import annotations

import torch

from . import _lib

__all__ = ["Reducer", "axpby", "colscale", "colscale_batched", "lincomb3"]


class Reducer:
    """Holds the partial-sum scratch; results land in a small device array and
    are fetched to the host in one copy when needed."""

    def __init__(self, device, max_k: int = _lib.MAX_MDOT):
        lib = _lib.lib()
        self.nb = int(lib.sgk_reduce_blocks())
        self.part = torch.empty(max_k * self.nb, dtype=torch.float64, device=device)
        self.max_k = max_k

    def dots(self, x: torch.Tensor, ys: torch.Tensor, out: torch.Tensor, sqrt: bool = False) -> torch.Tensor:
        """out[j] = x . ys[j] for ys of shape (k, n) (row stride = ys.stride(0))."""
        lib = _lib.lib()
        s = _lib.stream_ptr()
        k = ys.shape[0] if ys.dim() == 2 else 1
        n = x.numel()
        ystride = ys.stride(0) if ys.dim() == 2 else 0
        if k > self.max_k:
            raise ValueError("too many simultaneous dot products")
        _lib.check(lib.sgk_dot_partial(n, x.data_ptr(), ys.data_ptr(), ystride, k, self.part.data_ptr(), s),
                   "sgk_dot_partial")
        _lib.check(lib.sgk_reduce_partials(self.part.data_ptr(), k, out.data_ptr(), int(sqrt), s),
                   "sgk_reduce_partials")
        return out

    def dot(self, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        return self.dots(x.reshape(-1), y.reshape(1, -1), out)

    def norm(self, x: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        xf = x.reshape(-1)
        return self.dots(xf, xf.reshape(1, -1), out, sqrt=True)

    def mgs_step(self, dh: torch.Tensor, q: torch.Tensor, w: torch.Tensor, q_next: torch.Tensor | None,
                 out_next: torch.Tensor | None) -> None:
        """w -= (*dh) q ; then out_next = q_next . w (deterministic)."""
        lib = _lib.lib()
        s = _lib.stream_ptr()
        _lib.check(lib.sgk_mgs_step(w.numel(), dh.data_ptr(), q.data_ptr(), w.data_ptr(),
                                    q_next.data_ptr() if q_next is not None else None,
                                    self.part.data_ptr() if q_next is not None else None, s),
                   "sgk_mgs_step")
        if q_next is not None:
            _lib.check(lib.sgk_reduce_partials(self.part.data_ptr(), 1, out_next.data_ptr(), 0, s),
                       "sgk_reduce_partials")


def axpby(y: torch.Tensor, x: torch.Tensor | None, a: float = 1.0, b: float = 1.0,
          da: torch.Tensor | None = None, inv_a: bool = False, db: torch.Tensor | None = None) -> torch.Tensor:
    """y <- a*x + b*y where a may be scaled (or divided) by a device scalar."""
    lib = _lib.lib()
    _lib.check(lib.sgk_axpby_dev(y.numel(), a, da.data_ptr() if da is not None else None, int(inv_a),
                                 x.data_ptr() if x is not None else None, b,
                                 db.data_ptr() if db is not None else None, y.data_ptr(), _lib.stream_ptr()),
               "sgk_axpby_dev")
    return y


def lincomb3(out: torch.Tensor, x0: torch.Tensor, c1: float = 0.0, x1: torch.Tensor | None = None,
             c2: float = 0.0, x2: torch.Tensor | None = None, s: float = 1.0) -> torch.Tensor:
    """out <- s*((x0 + c1 x1) + c2 x2), bit-identical to the axpby chain
    (out = x0.clone(); axpby(out, x1, c1); axpby(out, x2, c2); axpby(out, None, 0, s))
    in one pass; `out` may be `x0`."""
    lib = _lib.lib()
    _lib.check(lib.sgk_lincomb3(out.numel(), x0.data_ptr(), c1, x1.data_ptr() if x1 is not None else None, c2,
                                x2.data_ptr() if x2 is not None else None, s, out.data_ptr(), _lib.stream_ptr()),
               "sgk_lincomb3")
    return out


def colscale_batched(x: torch.Tensor, w: torch.Tensor | None, s: torch.Tensor, out: torch.Tensor,
                     invert: bool = False):
    """out[b] = s[b] * (x[b] / w or x[b] * w) for a (n_b, n_rows, n_cols)
    stack; `s` a device vector of n_b scalars.  Per element the same
    arithmetic as `colscale`."""
    lib = _lib.lib()
    n_b, n_rows, n_cols = x.shape
    if s.numel() != n_b or not (x.is_contiguous() and out.is_contiguous()):
        raise ValueError("colscale_batched: need contiguous stacks and one scalar per block")
    _lib.check(lib.sgk_colscale_batched(n_b, n_rows, n_cols, x.data_ptr(), w.data_ptr() if w is not None else None,
                                        int(invert), s.data_ptr(), out.data_ptr(), _lib.stream_ptr()),
               "sgk_colscale_batched")
    return out


def colscale(x: torch.Tensor, w: torch.Tensor | None, s: float, out: torch.Tensor, invert: bool = False):
    lib = _lib.lib()
    n_rows, n_cols = x.shape
    _lib.check(lib.sgk_colscale(n_rows, n_cols, x.data_ptr(), w.data_ptr() if w is not None else None,
                                int(invert), s, out.data_ptr(), _lib.stream_ptr()), "sgk_colscale")
    return out
