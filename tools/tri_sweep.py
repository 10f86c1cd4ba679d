"""Time P~ / A~ solves for several widths (tuning helper)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system
cfg = int(sys.argv[1])
b = build_problem(cfg); s = steady_system(b)
soc = build_coupled_preconditioner(s, b.partition)
fac = soc.kkt_factor.device_factors
shape = (s.n_h, s.n_xi)
blk = [torch.randn(shape, dtype=torch.float64, device="cuda") for _ in range(3)]
out = [torch.empty_like(blk[0]) for _ in range(3)]
res = []
for lo, hi in b.partition.ranges():
    segs = [(t, lo) for t in blk]; o2 = [(t, lo) for t in out]
    fac.solve_segments(segs, o2, hi - lo); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): fac.solve_segments(segs, o2, hi - lo)
    e1.record(); e1.synchronize()
    res.append(f"w{hi-lo}:{e0.elapsed_time(e1)/3:.1f}")
print(os.environ.get("TAG", ""), " ".join(res), flush=True)
