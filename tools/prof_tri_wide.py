"""Driver for ncu: one config-5 P~ solve of the given width (wide-tiled path)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system
width = int(sys.argv[1]) if len(sys.argv) > 1 else 330
b = build_problem(5); s = steady_system(b)
fac = build_coupled_preconditioner(s, b.partition).kkt_factor.device_factors
blk = [torch.randn((s.n_h, width), dtype=torch.float64, device="cuda") for _ in range(3)]
out = [torch.empty_like(blk[0]) for _ in range(3)]
for _ in range(2):
    fac.solve_segments([(t, 0) for t in blk], [(t, 0) for t in out], width)
torch.cuda.synchronize()
print("width", width, "tiles L/U", fac.wl.n_tiles, fac.wu.n_tiles)
