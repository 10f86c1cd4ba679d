"""Time the config-4 matvec with the shipped library and with each variant
under build_variants/ named on the command line (A/B probes):
python tools/ab_variants.py gu4 gu8 ...   (name[:ENV=VAL,...])"""
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
ts = []
for rep in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])
    e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 10)
import hashlib
print("%%.4f ms (min %%.4f)  sha %%s" %% (sorted(ts)[2], min(ts), hashlib.sha1(w.cpu().numpy().tobytes()).hexdigest()[:10]))
''' % ROOT
for spec in ["shipped"] + sys.argv[1:]:
    name, _, envs = spec.partition(":")
    env = dict(os.environ)
    if name != "shipped":
        env["SGKKT_B200_LIB"] = str(ROOT / "build_variants" / f"libsgkkt_{name}.so")
    for kv in filter(None, envs.split(",")):
        k, _, v = kv.partition("=")
        env[k] = v
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"{spec:28s} {out.stdout.strip()} {out.stderr.strip()[-300:]}", flush=True)
