"""Host vs device time of one time-dependent preconditioner apply and KKT
apply (bench.py's time_solve_block setting: N=961, n_xi=20, 84 terms, N_t=8).
If the wall time per apply far exceeds the device time, the path is bound by
host launch overhead."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_23804_b200 import _lib
from paper_2512_23804_b200.problems import ConfigSpec, build_problem, steady_system
from paper_2512_23804_b200.timedep import (TimeKKT, build_time_preconditioner, build_time_stencil,
                                           time_kkt_apply_device, time_rhs, to_device_layout)

spec = ConfigSpec("time_paper", "control", 32, 3, 3, "hermite", "lognormal", 0.2, 1.0,
                  coefficient_degree=6, beta=1e-4, lo=-1.0, hi=1.0)
b = build_problem(spec, kl_method="dense")
st = steady_system(b)
sys_ = TimeKKT(steady=st, stencil=build_time_stencil(8), initial_state=np.zeros((st.n_h, st.n_xi)))
bd = to_device_layout(sys_, time_rhs(sys_))
out = torch.empty_like(bd)


def both(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    wall_enqueue = (time.perf_counter() - t0) / reps
    e1.synchronize()
    return wall_enqueue * 1e3, e0.elapsed_time(e1) / reps, (_lib.launch_count() - l0) / reps


for ls in ("lu", "fastdiag"):
    prec = build_time_preconditioner(sys_, b.partition, "cheb5", lead_solver=ls)
    w, g, n = both(lambda: prec.apply_device(bd, out))
    print(f"prec[{ls}] apply: host enqueue {w:.2f} ms, device {g:.2f} ms, {n:.0f} launches ({1e3 * w / max(n, 1):.1f} us each)")
w, g, n = both(lambda: time_kkt_apply_device(sys_, bd, out))
print(f"kkt apply: host enqueue {w:.2f} ms, device {g:.2f} ms, {n:.0f} launches")
from paper_2512_23804_b200.timedep import time_kkt_apply_interleaved

w, g, n = both(lambda: time_kkt_apply_interleaved(sys_, bd, out))
print(f"kkt apply (interleaved, one program): host enqueue {w:.2f} ms, device {g:.2f} ms, {n:.0f} launches")
