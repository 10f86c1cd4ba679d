"""Block-diagonal preconditioner apply and its A~_1 lead solves per lead
solver (lu / lu_nd / fastdiag) at one control configuration."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_23804_b200.preconditioners import build_steady_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


b = build_problem(cfg)
s = steady_system(b)
shape = (s.n_h, s.n_xi)
rng = np.random.default_rng(0)
blocks = [torch.as_tensor(rng.standard_normal(shape)).cuda() for _ in range(3)]
outs = tuple(torch.empty_like(blocks[0]) for _ in range(3))
for ls in ("lu", "lu_nd", "fastdiag"):
    bd = build_steady_preconditioner(s, b.partition, "cheb5", lead_solver=ls)
    f = bd.sweep.lead_factor.device_factors
    line = [f"{ls:9s} blockdiag apply {timed(lambda: bd.apply_device(*blocks, outs=outs)):.3f} ms |"]
    for lo, hi in b.partition.ranges():
        segs = [(outs[0], lo)]
        line.append(f"w{hi - lo}:{timed(lambda: f.solve_segments(segs, segs, hi - lo)):.3f}")
    extra = f" depth L/U {f.depth_l}/{f.depth_u} groups {f.gdepth_l}/{f.gdepth_u} nnz {f.nnz_l + f.nnz_u}" \
        if hasattr(f, "depth_l") else ""
    print(" ".join(line) + extra, flush=True)
