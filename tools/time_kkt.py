"""Config-5 KKT matvec: one 3-input launch vs the split (WS + mass) launches;
checked against each other and timed with CUDA events."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_23804_b200 import operators as ops
from paper_2512_23804_b200.problems import build_problem, steady_system
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
b = build_problem(cfg); s = steady_system(b)
shape = (s.n_h, s.n_xi)
rng = np.random.default_rng(0)
blk = [torch.as_tensor(rng.standard_normal(shape)).cuda() for _ in range(3)]
res = {}
for split in (False, True):
    ops.KKT_SPLIT = split
    out = tuple(torch.empty_like(blk[0]) for _ in range(3))
    fn = lambda: ops.steady_kkt_apply_device(s, *blk, out)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res[split] = ([o.clone() for o in out], ms)
    print(f"split={split}: {ms:.3f} ms  {s.algorithmic_bytes() / ms / 1e6:.0f} GB/s", flush=True)
err = max(float((a - c).abs().max() / c.abs().max()) for a, c in zip(res[True][0], res[False][0]))
print("max rel diff split vs fused:", err)
