"""ncu driver: three Chebyshev mass solves (cheb5, all columns) at config 5."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_23804_b200.preconditioners import build_steady_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system
b = build_problem(5); sys_ = steady_system(b)
bd = build_steady_preconditioner(sys_, b.partition, "cheb5", lead_solver="fastdiag")
x = torch.as_tensor(np.random.default_rng(0).standard_normal((sys_.n_h, sys_.n_xi))).cuda()
for _ in range(3):
    bd.mass_solve(x)
torch.cuda.synchronize()
print("done")
