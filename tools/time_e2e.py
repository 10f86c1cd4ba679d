"""Pinned-host end-to-end matvec (config 4): raw H2D / D2H copy rates and the
slab pipeline of operators._kron_apply_pipelined for several slab counts."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_23804_b200 import operators
from paper_2512_23804_b200.operators import KroneckerSumOperator
from paper_2512_23804_b200.problems import build_problem

b = build_problem(4)
op = KroneckerSumOperator(couplings=b.triple.matrices[: b.n_terms], operators=b.stiffness)
x = torch.from_numpy(np.random.default_rng(0).standard_normal((b.n_h, b.n_xi))).pin_memory()
w = torch.empty_like(x).pin_memory()
xd = torch.empty_like(x, device="cuda")
nbytes = x.numel() * 8


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


t = ev_time(lambda: xd.copy_(x, non_blocking=True))
print(f"H2D {nbytes / t / 1e6:.1f} GB/s ({t:.2f} ms)")
t = ev_time(lambda: w.copy_(xd, non_blocking=True))
print(f"D2H {nbytes / t / 1e6:.1f} GB/s ({t:.2f} ms)")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s1):
        xd.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        w.copy_(xd[:0].new_empty(0) if False else w.new_empty(0), non_blocking=True) if False else None
        w.copy_(torch.empty(0)) if False else None
    torch.cuda.current_stream().wait_stream(s1)


yd = torch.empty_like(xd)


def duplex():
    with torch.cuda.stream(s1):
        xd.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        w.copy_(yd, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t = ev_time(duplex)
print(f"H2D+D2H concurrent: {2 * nbytes / t / 1e6:.1f} GB/s total ({t:.2f} ms)")
for n in (8, 16, 32, 64, 128):
    t = ev_time(lambda: operators._kron_apply_pipelined(op, x, w, n_slabs=n))
    print(f"pipeline n_slabs={n}: {t:.2f} ms  {op.algorithmic_bytes() / t / 1e6:.1f} GB/s algorithmic", flush=True)
