"""Host vs device setup time: problems.build_problem
(SciPy assembly of every A_t, then the device layout upload on first use) vs
gpu_setup.build_problem_device, per BASELINE config."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_23804_b200.gpu_setup import build_problem_device
from paper_2512_23804_b200.operators import KroneckerSumOperator
from paper_2512_23804_b200.problems import build_problem

torch.zeros(1, device="cuda")
build_problem_device(1)  # warm the library / kernels
for cfg in [int(a) for a in sys.argv[1:]] or [3, 4, 5]:
    t0 = time.perf_counter()
    h = build_problem(cfg)
    op = KroneckerSumOperator(couplings=h.triple.matrices[: h.n_terms], operators=h.stiffness)
    op.pattern.pattern9()
    torch.cuda.synchronize()
    th = time.perf_counter() - t0
    t0 = time.perf_counter()
    d = build_problem_device(cfg)
    op = KroneckerSumOperator(couplings=d.triple.matrices[: d.n_terms], operators=d.stiffness)
    assert op.pattern is d.extras["device_pattern"]
    torch.cuda.synchronize()
    td = time.perf_counter() - t0
    print(f"cfg{cfg}: n_t={h.n_terms} host setup+upload {th:.2f} s, device setup {td:.2f} s "
          f"{ {k: round(v, 3) for k, v in d.extras['setup_seconds'].items()} }", flush=True)
