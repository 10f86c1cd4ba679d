"""Time the config-5 P~ triangular solves per RHS width (the hGSoc level
widths), grouped kernel vs wide-tiled kernel, checked against SuperLU; then
one hGSoc apply with LU leads."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import scipy.sparse.linalg as spla
from paper_2512_23804_b200 import linalg
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, deterministic_kkt_matrix
from paper_2512_23804_b200.problems import build_problem, steady_system
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
b = build_problem(cfg); s = steady_system(b)
t0 = time.perf_counter()
soc = build_coupled_preconditioner(s, b.partition)
fac = soc.kkt_factor.device_factors
print(f"setup {time.perf_counter() - t0:.1f} s; tiles L/U {fac.wl.n_tiles}/{fac.wu.n_tiles} slots {fac.wl_slots}/{fac.wu_slots}",
      flush=True)
n = s.n_h
lu = soc.kkt_factor._solver
rng = np.random.default_rng(0)
for width in (1, 8, 36, 64, 120, 330):
    rhs = rng.standard_normal((3 * n, width))
    segs = [torch.as_tensor(np.ascontiguousarray(rhs[i * n:(i + 1) * n])).cuda() for i in range(3)]
    outs = [torch.empty_like(x) for x in segs]
    res = {}
    for name, wmin in (("grouped", 10**9), ("wide", 32)):
        if name == "wide" and width < 32:
            continue
        linalg.WIDE_MIN = wmin
        for _ in range(2):
            fac.solve_segments([(x, 0) for x in segs], [(o, 0) for o in outs], width)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fac.solve_segments([(x, 0) for x in segs], [(o, 0) for o in outs], width)
            e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        got = np.concatenate([o.cpu().numpy() for o in outs])
        res[name] = (float(np.median(ts)), got)
    want = lu.solve(rhs)
    line = f"width {width:4d}:"
    for name, (ms, got) in res.items():
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        line += f"  {name} {ms:8.3f} ms (rel err {err:.1e})"
    if len(res) == 2:
        line += f"  bitwise-equal {np.array_equal(res['grouped'][1], res['wide'][1])}"
    print(line, flush=True)
linalg.WIDE_MIN = 32
r = [torch.randn((n, s.n_xi), dtype=torch.float64, device="cuda") for _ in range(3)]
o = [torch.empty_like(x) for x in r]
for wmin, name in ((10**9, "grouped"), (32, "wide")):
    linalg.WIDE_MIN = wmin
    soc.apply_device(*r, outs=tuple(o)); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        soc.apply_device(*r, outs=tuple(o))
    e1.record(); torch.cuda.synchronize()
    print(f"hGSoc apply (LU, {name} wide solves): {e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
