"""Speed-of-light probes of the config-4 WS matvec kernel: time the normal
kernel against debug builds (build_variants/) that truncate the producers'
step loop or the consumers' gather (results intentionally wrong)."""
import os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, "%s")
from paper_2512_23804_b200.device import run_program
from paper_2512_23804_b200.operators import KroneckerSumOperator
from paper_2512_23804_b200.problems import build_problem
b = build_problem(4)
op = KroneckerSumOperator(couplings=b.triple.matrices[: b.n_terms], operators=b.stiffness)
x = torch.as_tensor(np.random.default_rng(0).standard_normal((b.n_h, b.n_xi))).cuda()
w = torch.empty_like(x)
prog = op.program([(0, b.n_xi)], (0, b.n_xi), 0, op.n_terms)
for _ in range(3): run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
e1.record(); torch.cuda.synchronize()
print("%%.4f" %% (e0.elapsed_time(e1) / 20))
''' % ROOT
for name in ("normal", "halfsteps", "noprod", "nogather", "halfgather"):
  for grid in ("0", "1"):
    env = dict(os.environ)
    env["SGKKT_GRID9"] = grid
    if name != "normal":
        env["SGKKT_B200_LIB"] = str(ROOT / "build_variants" / f"libsgkkt_{name}.so")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"{name:10s} grid={grid} {out.stdout.strip()} ms {out.stderr.strip()[-200:]}", flush=True)
