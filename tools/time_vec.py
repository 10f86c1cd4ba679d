"""HBM bandwidth of the Krylov vector kernels (deterministic dots, fused MGS
step, axpby) on config-5-sized vectors (3 x 16129 x 495 doubles = 192 MB)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_23804_b200.vec import Reducer, axpby

n = 3 * 16129 * 495
dev = torch.device("cuda")
x, y, z = (torch.randn(n, dtype=torch.float64, device=dev) for _ in range(3))
red = Reducer(dev)
out = torch.zeros(8, dtype=torch.float64, device=dev)
basis = torch.randn((8, n), dtype=torch.float64, device=dev)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for name, fn, nbytes in (
    ("dot (2 reads)", lambda: red.dot(x, y, out[0:1]), 16 * n),
    ("norm (1 read)", lambda: red.norm(x, out[0:1]), 8 * n),
    ("dots x.basis[0:8] (9 reads)", lambda: red.dots(x, basis, out), 72 * n),
    ("mgs_step (3 reads + 1 write)", lambda: red.mgs_step(out[0:1], y, z, x, out[1:2]), 32 * n),
    ("axpby (2 reads + 1 write)", lambda: axpby(y, x, 0.5, 1.0), 24 * n),
):
    ms = timed(fn)
    print(f"{name:32s} {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s", flush=True)
