"""Row-slab sharded Galerkin matvec across GPUs.

One process per GPU (`torch.distributed`, NCCL on the GPUs; gloo in the CPU
tests).  The mesh rows are cut into contiguous slabs, one per rank; a rank
owns the rows [a, b) of V and W.  The 9-point stencil of a row reaches at most
`reach` rows away (m + 1 on an m x m grid), so before each matvec a rank
receives the last `reach` owned rows of its left neighbour and the first
`reach` of its right neighbour (one send/recv pair per side: the only
exchange step — about 2 x (m+1) x n_xi doubles, 4 MB per side at config 4)
and runs the coupling kernel on its own rows (`run_program(rows=(a, b))`).
The chaos-space couplings H_t need no exchange (every rank holds all of them).

The halo logic is plain host code (`slab_rows`, `halo_ranges`,
`exchange_halo`) and is tested with gloo, world size 2, on the CPU
(tests/test_sharded.py); the device part is the row-range launch of the
single-GPU kernel.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["ShardedKron", "exchange_halo", "halo_ranges", "slab_rows", "stencil_reach"]


def slab_rows(n_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row slab [a, b) of `rank`."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    edges = np.linspace(0, n_rows, world + 1).round().astype(np.int64)
    return int(edges[rank]), int(edges[rank + 1])


def stencil_reach(indptr: np.ndarray, indices: np.ndarray) -> int:
    """Largest |column - row| of the pattern (m + 1 on an m x m 9-point grid)."""
    n = len(indptr) - 1
    rows = np.repeat(np.arange(n), np.diff(indptr))
    return int(np.abs(indices - rows).max()) if len(indices) else 0


def halo_ranges(n_rows: int, world: int, rank: int, reach: int):
    """(left, right) halo row ranges a rank receives, and (left, right) owned
    row ranges it sends; empty ranges at the ends.  Requires every slab to be
    at least `reach` rows (the halo comes from the direct neighbours only)."""
    a, b = slab_rows(n_rows, world, rank)
    if world > 1 and min(slab_rows(n_rows, world, r)[1] - slab_rows(n_rows, world, r)[0]
                         for r in range(world)) < reach:
        raise ValueError("slabs thinner than the stencil reach: use fewer ranks")
    recv_left = (max(0, a - reach), a) if rank > 0 else (a, a)
    recv_right = (b, min(n_rows, b + reach)) if rank < world - 1 else (b, b)
    send_left = (a, min(b, a + reach)) if rank > 0 else (a, a)
    send_right = (max(a, b - reach), b) if rank < world - 1 else (b, b)
    return recv_left, recv_right, send_left, send_right


def exchange_halo(v_full: torch.Tensor, n_rows: int, reach: int, group=None) -> None:
    """Fill the halo rows of this rank's full-height buffer from its
    neighbours (owned rows must already be in place)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return
    rl, rr, sl, sr = halo_ranges(n_rows, world, rank, reach)
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, v_full[sl[0]:sl[1]].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, v_full[rl[0]:rl[1]], rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, v_full[sr[0]:sr[1]].contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, v_full[rr[0]:rr[1]], rank + 1, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()


class ShardedKron:
    """W[a:b] = (sum_t A_t V H_t)[a:b] on this rank's slab, V given by its owned
    rows; `apply` exchanges the halo and launches the 9-point coupling kernel
    on the owned rows (the operator's full pattern lives on every rank)."""

    def __init__(self, op, group=None):
        self.op = op
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        pat = op.pattern
        self.n_rows = pat.n_rows
        self.reach = stencil_reach(pat.indptr, pat.indices)
        self.rows = slab_rows(self.n_rows, self.world, self.rank)
        if pat.pattern9() is None:
            raise ValueError("the sharded matvec needs the 9-point fast path")
        n_xi = op.shape[1]
        self.prog = op.program([(0, n_xi)], (0, n_xi), 0, op.n_terms)
        self.v_full = torch.zeros((self.n_rows, n_xi), dtype=torch.float64, device=pat._vals.device)
        self.w_full = torch.empty_like(self.v_full)

    def apply(self, v_owned: torch.Tensor) -> torch.Tensor:
        from .device import run_program

        a, b = self.rows
        if tuple(v_owned.shape) != (b - a, self.op.shape[1]):
            raise ValueError("owned block has the wrong shape")
        self.v_full[a:b].copy_(v_owned)
        if self.world > 1:  # NCCL orders its sends after the copy (current-stream dependency)
            exchange_halo(self.v_full, self.n_rows, self.reach, self.group)
        run_program(self.op.pattern, self.prog, [(self.v_full, 0)], [(self.w_full, 0)], alpha=[1.0], beta=[0.0],
                    rows=(a, b))
        return self.w_full[a:b]
