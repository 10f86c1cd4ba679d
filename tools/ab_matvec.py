"""A/B the config-4 matvec kernels: the grid kernel (sliding V window,
contiguous row ranges) against the pattern-indexed warp-specialised kernel;
checks bitwise agreement and times both with CUDA events (median of reps)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_23804_b200 import device as dev
from paper_2512_23804_b200.device import run_program
from paper_2512_23804_b200.operators import KroneckerSumOperator
from paper_2512_23804_b200.problems import build_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
b = build_problem(cfg)
op = KroneckerSumOperator(couplings=b.triple.matrices[: b.n_terms], operators=b.stiffness)
x = torch.as_tensor(np.random.default_rng(0).standard_normal((b.n_h, b.n_xi))).cuda()
prog = op.program([(0, b.n_xi)], (0, b.n_xi), 0, op.n_terms)
flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")


def run(grid, reps=30):
    dev.GRID9 = grid
    w = torch.empty_like(x)
    for _ in range(3):
        run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return w, float(np.median(ts)), float(np.min(ts))


B = op.algorithmic_bytes()
import os
for seg in (8, 17, 32, 64, 128, 255):
    os.environ["SGKKT_GRID_SEG"] = str(seg)
    w_, m_, b_ = run(True)
    print(f"grid seg {seg}: median {m_:.4f} ms best {b_:.4f} ms  {B / m_ / 1e6:.0f} GB/s", flush=True)
del os.environ["SGKKT_GRID_SEG"]
wg, mg, bg = run(True)
ww, mw, bw = run(False)
print(f"grid: median {mg:.4f} ms best {bg:.4f} ms  {B / mg / 1e6:.0f} GB/s")
print(f"ws  : median {mw:.4f} ms best {bw:.4f} ms  {B / mw / 1e6:.0f} GB/s")
print("bitwise equal:", torch.equal(wg, ww), "max rel diff", float((wg - ww).abs().max() / ww.abs().max()))
