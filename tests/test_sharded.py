"""Row-slab sharding of the Galerkin matvec: slab/halo host
logic and the halo exchange with gloo, world size 2, on the CPU (the
exchanged rows + the oracle reproduce the global matvec rows); on the GPU
the row-range kernel launches with only owned + halo rows valid (the rest
NaN) reproduce the single-launch matvec."""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def test_slabs_and_halo_ranges():
    from paper_2512_23804_b200.sharded import halo_ranges, slab_rows

    n, world, reach = 100, 4, 11
    slabs = [slab_rows(n, world, r) for r in range(world)]
    assert slabs[0][0] == 0 and slabs[-1][1] == n
    assert all(slabs[r][1] == slabs[r + 1][0] for r in range(world - 1))
    for r in range(world):
        rl, rr, sl, sr = halo_ranges(n, world, r, reach)
        a, b = slabs[r]
        assert rl[1] == a and rr[0] == b
        assert (rl[1] - rl[0]) == (0 if r == 0 else reach) and (rr[1] - rr[0]) == (0 if r == world - 1 else reach)
        # what I send left is what my left neighbour receives on its right
        if r > 0:
            assert sl == halo_ranges(n, world, r - 1, reach)[1]
    with pytest.raises(ValueError):
        halo_ranges(20, 4, 11, 11)


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2512_23804_b200.problems import build_problem
    from paper_2512_23804_b200.sharded import exchange_halo, slab_rows, stencil_reach

    b = build_problem(1, n=12)
    cp = b.triple.matrices[: b.n_terms]
    a_mat = b.stiffness[0].tocsr()
    reach = stencil_reach(a_mat.indptr, a_mat.indices)
    v_global = np.random.default_rng(5).standard_normal((b.n_h, b.n_xi))
    lo, hi = slab_rows(b.n_h, world, rank)
    v_full = torch.full((b.n_h, b.n_xi), float("nan"), dtype=torch.float64)
    v_full[lo:hi] = torch.as_tensor(v_global[lo:hi])
    exchange_halo(v_full, b.n_h, reach)
    got = oracle.kron_apply_rows(cp, b.stiffness, np.nan_to_num(v_full.numpy(), nan=1e300), (lo, hi))
    want = oracle.kron_apply(cp, b.stiffness, v_global)[lo:hi]
    out[rank] = float(np.abs(got - want).max() / np.abs(want).max())
    dist.destroy_process_group()


def test_halo_exchange_gloo_reproduces_global_matvec():
    port = 29700 + os.getpid() % 1000
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] <= 1e-13 and out[1] <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_row_slab_launches_match_full_matvec(world):
    import torch

    from paper_2512_23804_b200.device import run_program
    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply
    from paper_2512_23804_b200.problems import build_problem
    from paper_2512_23804_b200.sharded import halo_ranges, slab_rows, stencil_reach

    b = build_problem(2)
    op = KroneckerSumOperator(couplings=b.triple.matrices[: b.n_terms], operators=b.stiffness)
    v = torch.as_tensor(np.random.default_rng(6).standard_normal((b.n_h, b.n_xi))).cuda()
    want = kron_apply(op, v)
    reach = stencil_reach(op.pattern.indptr, op.pattern.indices)
    prog = op.program([(0, b.n_xi)], (0, b.n_xi), 0, op.n_terms)
    for r in range(world):
        lo, hi = slab_rows(b.n_h, world, r)
        rl, rr, _, _ = halo_ranges(b.n_h, world, r, reach)
        v_full = torch.full_like(v, float("nan"))
        v_full[rl[0]:rr[1]] = v[rl[0]:rr[1]]  # owned + halo rows only
        w = torch.full_like(v, float("nan"))
        run_program(op.pattern, prog, [(v_full, 0)], [(w, 0)], alpha=[1.0], beta=[0.0], rows=(lo, hi))
        assert torch.equal(w[lo:hi], want[lo:hi])
