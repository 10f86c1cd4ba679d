"""Config-4 matvec with contiguous states (row stride n_xi = 1001 doubles: rows
start on 8-byte boundaries) against states whose row stride is padded to a
multiple of 16 doubles (1008: every row starts on a 128-byte line)."""
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
x0 = torch.as_tensor(np.random.default_rng(0).standard_normal((b.n_h, b.n_xi))).cuda()
prog = op.program([(0, b.n_xi)], (0, b.n_xi), 0, op.n_terms)
ref = None
for pad in (0, 16, 2):
    ld = b.n_xi if pad == 0 else (b.n_xi + pad - 1) // pad * pad
    xs = torch.zeros((b.n_h, ld), dtype=torch.float64, device="cuda")
    ws = torch.zeros((b.n_h, ld), dtype=torch.float64, device="cuda")
    x, w = xs[:, : b.n_xi], ws[:, : b.n_xi]
    x.copy_(x0)
    for _ in range(3):
        run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
    torch.cuda.synchronize()
    ts = []
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 10)
    if ref is None:
        ref = w.clone()
    same = bool(torch.equal(ref, w))
    print(f"cfg{cfg} row stride {ld}: {sorted(ts)[2]:.4f} ms (min {min(ts):.4f})  bit-equal to contiguous: {same}", flush=True)
