"""Minimal driver for ncu: build cfg4 and run a few Galerkin matvecs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_23804_b200.device import run_program
from paper_2512_23804_b200.operators import KroneckerSumOperator
from paper_2512_23804_b200.problems import build_problem

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
b = build_problem(cfg)
op = KroneckerSumOperator(couplings=b.triple.matrices[: b.n_terms], operators=b.stiffness)
x = torch.as_tensor(np.random.default_rng(0).standard_normal((b.n_h, b.n_xi))).cuda()
w = torch.empty_like(x)
prog = op.program([(0, b.n_xi)], (0, b.n_xi), 0, op.n_terms)
for _ in range(reps):
    run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
torch.cuda.synchronize()
print("done", prog.host.stats)
