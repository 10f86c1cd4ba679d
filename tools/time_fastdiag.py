"""Per-piece CUDA-event timings of the fast-diagonalisation solve path
 at one control configuration:

    python tools/time_fastdiag.py [cfg] [beta]

KKT matvec, one hGSoc apply (couplings vs P~ solves per level), one
block-diagonal apply (Chebyshev mass solves, hGS sweep, A~ solves), and the
achieved fp64 rate of the DGEMM passes (24 w n^3 flops per P~ solve of width w,
8 w n^3 per lead solve)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_23804_b200.device import run_program
from paper_2512_23804_b200.operators import steady_kkt_apply_device
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, build_steady_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
beta = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


b = build_problem(cfg, beta=beta)
sys_ = steady_system(b)
shape = (sys_.n_h, sys_.n_xi)
n = int(round(np.sqrt(sys_.n_h)))
rng = np.random.default_rng(0)
blocks = [torch.as_tensor(rng.standard_normal(shape)).cuda() for _ in range(3)]
outs = tuple(torch.empty_like(blocks[0]) for _ in range(3))
print(f"cfg{cfg} beta={beta} N={b.n_h} (n={n}) n_xi={b.n_xi} n_t={b.n_terms}")
print(f"kkt matvec {timed(lambda: steady_kkt_apply_device(sys_, *blocks, outs)):.3f} ms")
soc = build_coupled_preconditioner(sys_, b.partition, lead_solver="fastdiag")
fac = soc.kkt_factor
print(f"hgsoc[fastdiag] apply {timed(lambda: soc.apply_device(*blocks, outs=outs)):.3f} ms")
fwd, bwd = soc._programs()
pat = sys_.pattern
tot_c = tot_s = 0.0
ranges = b.partition.ranges()
for (lo, hi), prog in list(zip(ranges, fwd)) + list(zip(reversed(ranges[:-1]), bwd)):
    ins = [(o, 0) for o in outs]
    dst = [(o, lo) for o in outs]
    init = [(r, lo) for r in blocks]
    tc = timed(lambda: run_program(pat, prog, ins, dst, init, alpha=[1.0] * 3, beta=[1.0] * 3))
    segs = [(o, lo) for o in outs]
    ts = timed(lambda: fac.solve_segments(segs, segs, hi - lo))
    w = hi - lo
    tf = 24.0 * w * n ** 3 / (ts * 1e-3) / 1e12
    print(f"  level width {w:4d}: coupling {tc:.3f} ms  P~ solve {ts:.3f} ms ({tf:.1f} fp64 TFLOP/s in the passes)")
    tot_c += tc
    tot_s += ts
print(f"  sum: couplings {tot_c:.3f} ms, P~ solves {tot_s:.3f} ms")
bd = build_steady_preconditioner(sys_, b.partition, "cheb5", lead_solver="fastdiag")
print(f"blockdiag[fastdiag] apply {timed(lambda: bd.apply_device(*blocks, outs=outs)):.3f} ms")
print(f"  mass solve (cheb5, all columns) {timed(lambda: bd.mass_solve(blocks[0])):.3f} ms")
print(f"  schur apply (2 hGS sweeps + weighted mass) {timed(lambda: bd.schur_apply_device(blocks[2])):.3f} ms")
print(f"  hgs sweep {timed(lambda: bd.sweep.apply_device(blocks[2])):.3f} ms")
lead = bd.sweep.lead_factor
for lo, hi in ranges:
    segs = [(outs[0], lo)]
    ts = timed(lambda: lead.solve_segments(segs, segs, hi - lo))
    print(f"  A~ solve width {hi - lo:4d}: {ts:.3f} ms ({8.0 * (hi - lo) * n ** 3 / (ts * 1e-3) / 1e12:.1f} TFLOP/s)")
# stacked segments (one Krylov vector's y/u/lambda blocks): passes 1 and 4 as one batch
stack = torch.empty((3, sys_.n_h, sys_.n_xi), dtype=torch.float64, device="cuda")
sb = [stack[i] for i in range(3)]
tot = 0.0
for lo, hi in ranges:
    segs = [(t_, lo) for t_ in sb]
    tot += timed(lambda: fac.solve_segments(segs, segs, hi - lo))
sep = 0.0
for lo, hi in ranges:
    segs = [(t_, lo) for t_ in outs]
    sep += timed(lambda: fac.solve_segments(segs, segs, hi - lo))
print(f"P~ solves over the 5 levels: separate segments {sep:.3f} ms, stacked segments {tot:.3f} ms")
