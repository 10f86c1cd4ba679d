"""Minimal ncu driver: the hGSoc coupling launch of one degree level
(config 5 by default, the forward widest level)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_23804_b200.device import run_program
from paper_2512_23804_b200.preconditioners import CoupledSweepPreconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
level = int(sys.argv[2]) if len(sys.argv) > 2 else -1
b = build_problem(cfg)
s = steady_system(b)
soc = CoupledSweepPreconditioner(system=s, partition=b.partition, n_tau=s.n_terms, kkt_factor=None)
fwd, _ = soc._programs()
lo, hi = b.partition.ranges()[level]
prog = fwd[level]
rng = np.random.default_rng(0)
blocks = [torch.as_tensor(rng.standard_normal((s.n_h, s.n_xi))).cuda() for _ in range(3)]
outs = [torch.empty_like(blocks[0]) for _ in range(3)]
for _ in range(3):
    run_program(s.pattern, prog, [(o, 0) for o in blocks], [(o, lo) for o in outs], [(r, lo) for r in blocks],
                alpha=[1.0] * 3, beta=[1.0] * 3)
torch.cuda.synchronize()
print("done", prog.fast9(s.pattern.n_slices).host.stats)
