"""Phase anatomy of the config-4 warp-specialised matvec kernel (trace build:
`make s9trace` -> build_variants/libsgkkt_s9trace.so).  CTA 0 stamps clock64()
per mesh row: producer warps 0 and 7 — 0 row start, 1 after the producer
barrier, 2 after the EMPTY wait, 3 V registers arrived, 4 products stored,
5 next row's V loads issued; consumer warp 8 — 0 before FULL, 1 after FULL,
2 gather done.  Prints per-phase medians in SM cycles."""
import ctypes, os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
os.environ.setdefault("SGKKT_B200_LIB", str(ROOT / "build_variants" / "libsgkkt_s9trace.so"))
sys.path.insert(0, str(ROOT))
import numpy as np, torch
from paper_2512_23804_b200 import _lib
from paper_2512_23804_b200.device import run_program
from paper_2512_23804_b200.operators import KroneckerSumOperator
from paper_2512_23804_b200.problems import build_problem
b = build_problem(4)
op = KroneckerSumOperator(couplings=b.triple.matrices[: b.n_terms], operators=b.stiffness)
x = torch.as_tensor(np.random.default_rng(0).standard_normal((b.n_h, b.n_xi))).cuda()
w = torch.empty_like(x)
prog = op.program([(0, b.n_xi)], (0, b.n_xi), 0, op.n_terms)
for _ in range(3):
    run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
torch.cuda.synchronize()
lib = _lib.lib()
lib.sgk_s9_trace_read.argtypes = [ctypes.c_void_p]
arr = np.zeros((3, 256, 8), np.int64)
lib.sgk_s9_trace_read(arr.ctypes.data)
t = arr.astype(np.float64)
rows = slice(8, 250)
for w_, name in ((0, "producer warp 0"), (1, "producer warp 7")):
    p = t[w_, rows]
    period = np.median(np.diff(t[w_, rows, 0]))
    print(f"{name}: row period {period:.0f} clk")
    for a, bb, lab in ((0, 1, "wait_group + producer barrier"), (1, 2, "stage + EMPTY wait"), (2, 3, "V registers arrive"),
                       (3, 4, "products (11 steps)"), (4, 5, "FULL arrive + issue next V loads")):
        d = p[:, bb] - p[:, a]
        print(f"   {lab:34s} median {np.median(d):7.0f}  p10 {np.percentile(d, 10):7.0f}  p90 {np.percentile(d, 90):7.0f}")
c = t[2, rows]
print(f"consumer warp 8: row period {np.median(np.diff(t[2, rows, 0])):.0f} clk")
for a, bb, lab in ((0, 1, "wait FULL"), (1, 2, "gather + store")):
    d = c[:, bb] - c[:, a]
    print(f"   {lab:34s} median {np.median(d):7.0f}  p10 {np.percentile(d, 10):7.0f}  p90 {np.percentile(d, 90):7.0f}")
