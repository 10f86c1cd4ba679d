"""Driver for ncu: one wide P~ solve at config 5 (the top degree level)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
b = build_problem(cfg); s = steady_system(b)
fac = build_coupled_preconditioner(s, b.partition).kkt_factor.device_factors
lo, hi = b.partition.ranges()[int(sys.argv[2]) if len(sys.argv) > 2 else -1]
blk = [torch.randn((s.n_h, s.n_xi), dtype=torch.float64, device="cuda") for _ in range(3)]
out = [torch.empty_like(blk[0]) for _ in range(3)]
for _ in range(2):
    fac.solve_segments([(t, lo) for t in blk], [(t, lo) for t in out], hi - lo)
torch.cuda.synchronize()
print("width", hi - lo)
print("n", fac.n, "group depth L/U", fac.gdepth_l, fac.gdepth_u, "groups L/U", fac.gl.n_groups, fac.gu.n_groups,
      "nnz strict L/U", int(fac.gl_bufs[0][-1].item()), int(fac.gu_bufs[0][-1].item()))
