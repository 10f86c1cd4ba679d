"""Time the hot-path pieces of one configuration on the GPU (CUDA events)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_23804_b200.operators import steady_kkt_apply_device
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, build_steady_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
beta = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2


def timed(fn, reps=3):
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


t0 = time.time()
b = build_problem(cfg, beta=beta)
sys_ = steady_system(b)
print(f"cfg{cfg} beta={beta} build {time.time() - t0:.1f}s  N={b.n_h} n_xi={b.n_xi} n_t={b.n_terms}", flush=True)
shape = (sys_.n_h, sys_.n_xi)
rng = np.random.default_rng(0)
blocks = [torch.as_tensor(rng.standard_normal(shape)).cuda() for _ in range(3)]
outs = tuple(torch.empty_like(blocks[0]) for _ in range(3))
print(f"kkt matvec {timed(lambda: steady_kkt_apply_device(sys_, *blocks, outs)):.3f} ms", flush=True)
t0 = time.time()
soc = build_coupled_preconditioner(sys_, b.partition)
fac = soc.kkt_factor.device_factors
print(f"P~ factor+upload {time.time() - t0:.1f}s  nnzL={fac.nnz_l} nnzU={fac.nnz_u} depthL={fac.depth_l} depthU={fac.depth_u}", flush=True)
print(f"hgsoc apply {timed(lambda: soc.apply_device(*blocks, outs=outs), reps=2):.3f} ms", flush=True)
for lo, hi in b.partition.ranges():
    segs = [(blocks[0], lo), (blocks[1], lo), (blocks[2], lo)]
    o2 = [(outs[0], lo), (outs[1], lo), (outs[2], lo)]
    print(f"  P~ solve width {hi - lo}: {timed(lambda: fac.solve_segments(segs, o2, hi - lo), reps=2):.3f} ms", flush=True)
t0 = time.time()
bd = build_steady_preconditioner(sys_, b.partition, "cheb5")
lead = bd.sweep.lead_factor.device_factors
print(f"A~ factor+upload {time.time() - t0:.1f}s nnzL={lead.nnz_l} depthL={lead.depth_l} depthU={lead.depth_u}", flush=True)
print(f"blockdiag apply {timed(lambda: bd.apply_device(*blocks, outs=outs), reps=2):.3f} ms", flush=True)
print(f"hgs sweep {timed(lambda: bd.sweep.apply_device(blocks[2]), reps=2):.3f} ms", flush=True)
cheb = bd.mass_solve if hasattr(bd, "mass_solve") else None
for lo, hi in b.partition.ranges():
    segs = [(blocks[0], lo)]
    o2 = [(outs[0], lo)]
    print(f"  A~ solve width {hi - lo}: {timed(lambda: lead.solve_segments(segs, o2, hi - lo), reps=2):.3f} ms", flush=True)
print(f"  A~ dense regions: L {lead.gl.dense_nb} blocks, U {lead.gu.dense_nb} blocks; groups L/U {lead.gl.n_groups}/{lead.gu.n_groups}")
