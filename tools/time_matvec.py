"""Time the Galerkin matvec (cfg4 by default) with CUDA events.
`python tools/time_matvec.py 4 probe` also times a diagnostic run where every
row reads the same 9 input rows (L1-resident V: isolates the SM-side cost)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_23804_b200.device import run_program
from paper_2512_23804_b200.operators import KroneckerSumOperator
from paper_2512_23804_b200.problems import build_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
b = build_problem(cfg)
op = KroneckerSumOperator(couplings=b.triple.matrices[: b.n_terms], operators=b.stiffness)
x = torch.as_tensor(np.random.default_rng(0).standard_normal((b.n_h, b.n_xi))).cuda()
w = torch.empty_like(x)
prog = op.program([(0, b.n_xi)], (0, b.n_xi), 0, op.n_terms)


def timed(reps=20):
    for _ in range(3):
        run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = timed()
print(f"cfg{cfg} matvec {ms:.3f} ms {op.algorithmic_bytes() / ms / 1e6:.0f} GB/s  {prog.host.stats}", flush=True)
if len(sys.argv) > 2 and sys.argv[2] == "probe":
    pat = op.pattern
    pat.pattern9()
    saved = pat._colind9.clone()
    pat._colind9.copy_(torch.arange(9, dtype=torch.int32, device="cuda").repeat(pat.n_rows, 1).reshape(saved.shape))
    print(f"probe (V rows L1-resident): {timed(10):.3f} ms")
    pat._colind9.copy_(saved)
