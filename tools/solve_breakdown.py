"""Split a GPU hGSoc-FGMRES / MINRES solve into preconditioner, operator and
Krylov (rest) time (synchronising around the callables)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_23804_b200.krylov import FgmresConfig, fgmres, minres
from paper_2512_23804_b200.operators import steady_kkt_apply_device
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, build_steady_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system

cfg = int(sys.argv[1]); beta = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
b = build_problem(cfg, beta=beta); s = steady_system(b)
n = s.block_size(); shape = (s.n_h, s.n_xi)
rhs = np.zeros(3 * n); rhs[:n] = np.asarray(s.mass @ s.target).ravel()
bt = torch.as_tensor(rhs).cuda()
split = lambda v: [v[i * n:(i + 1) * n].view(shape) for i in range(3)]
acc = {"op": 0.0, "prec": 0.0}
def timed(key, fn):
    def f(v):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        o = fn(v); torch.cuda.synchronize(); acc[key] += time.perf_counter() - t0
        return o
    return f
def op(v):
    o = torch.empty_like(v); steady_kkt_apply_device(s, *split(v), tuple(split(o))); return o
for name, prec, solver in (("hgsoc_fgmres", build_coupled_preconditioner(s, b.partition), fgmres),
                           ("bd_minres", build_steady_preconditioner(s, b.partition, "cheb5"), minres)):
    def pr(v, prec=prec):
        o = torch.empty_like(v); prec.apply_device(*split(v), outs=tuple(split(o))); return o
    pr(bt); torch.cuda.synchronize()
    for rep in range(2):
        acc["op"] = acc["prec"] = 0.0
        torch.cuda.synchronize(); t0 = time.perf_counter()
        x, rep_ = solver(timed("op", op), timed("prec", pr), bt, FgmresConfig(tol=1e-8))
        torch.cuda.synchronize(); tt = time.perf_counter() - t0
    print(f"cfg{cfg} beta={beta} {name}: its={rep_.iterations} total={tt*1e3:.1f} ms prec={acc['prec']*1e3:.1f} op={acc['op']*1e3:.1f} rest={(tt-acc['prec']-acc['op'])*1e3:.1f}", flush=True)
