"""P~ triangular-solve times of SuperLU factors with different diagonal
pivot thresholds (the reference uses 1.0: partial pivoting)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import scipy.sparse.linalg as spla
import torch

from paper_2512_23804_b200.linalg import TriangularFactors
from paper_2512_23804_b200.preconditioners import deterministic_kkt_matrix
from paper_2512_23804_b200.problems import build_problem, steady_system

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
b = build_problem(cfg)
s = steady_system(b)
K = deterministic_kkt_matrix(s).tocsc()
shape = (s.n_h, s.n_xi)
blk = [torch.randn(shape, dtype=torch.float64, device="cuda") for _ in range(3)]
out = [torch.empty_like(blk[0]) for _ in range(3)]
for thr in (1.0, 0.1, 0.01):
    lu = spla.splu(K, diag_pivot_thresh=thr)
    fac = TriangularFactors.from_superlu(lu)
    res = []
    tot = 0.0
    for lo, hi in b.partition.ranges():
        segs = [(t, lo) for t in blk]
        o2 = [(t, lo) for t in out]
        fac.solve_segments(segs, o2, hi - lo)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fac.solve_segments(segs, o2, hi - lo)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 3
        tot += ms * (2 if hi - lo < b.n_xi - b.partition.ranges()[-1][0] else 1)
        res.append(f"w{hi - lo}:{ms:.1f}")
    print(f"thresh {thr}: depth L/U {fac.gdepth_l}/{fac.gdepth_u} nnz {fac.nnz_l + fac.nnz_u} " + " ".join(res)
          + f"  (sum over an hGSoc apply {tot:.1f} ms)", flush=True)
