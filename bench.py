#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric: "Galerkin matvec GB/s
vs HBM peak; hGSoc-MINRES time-to-solution + iterations").

Headline line (one JSON object on rank 0):
  * workload = BASELINE config 4 (the matvec stress test: N=65025, n_xi=1001,
    n_t=11, V ~ N(0,1) seeded, 520 MB > L2 so every timed matvec streams HBM);
  * a "step" = one Galerkin matvec W = sum_t A_t V H_t over the whole V;
  * value = algorithmic GB/s = B / t, B = 16 N n_xi + 8 n_t nnz(A)
    + 4 (nnz(A)+N+1) + 12 sum nnz(H_t)  (1095.3 MB at cfg4),
    whole job over all ranks (weak scaling: each rank its own matvecs);
  * e2e = same metric through the public drop-in API `kron_apply` with V in
    pinned host memory: H2D(V) + kernel + D2H(W) inside the timed region;
  * roofline = the matvec kernel (stencil9_kernel on the Q1 pattern) vs the
    measured HBM copy peak, plus its FP64 rate vs the measured DFMA peak (the
    kernel's binding pipe: 7.9 GFLOP per matvec);
  * cpu_baseline = the NumPy/SciPy oracle port of the reference path on a
    bounded row sample of the same workload, on this host;
  * solves = time-to-solution + iterations for config 2 (hGSoc-FGMRES and
    block-diagonal-hGS MINRES, tol 1e-8) — and config 5 with --solve-cfg5.

`--impl reference` times the oracle port (the reference is pure Python /
SciPy; there is no compiled reference) on the same metric.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
FP64_PEAK_TFLOPS = 36.4  # measured DFMA peak on this pool's B200 (tools/fp64_probe.cu; DMMA 37.1)
sys.path.insert(0, str(ROOT))

SEED = 20240817


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded or sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[3]) for r in rows if _isnum(r[3])), default=None)}


def _isnum(s):
    try:
        float(s)
        return True
    except ValueError:
        return False


def matvec_bytes(n_h, n_xi, n_t, nnz_a, nnz_h):
    return 16 * n_h * n_xi + 8 * n_t * nnz_a + 4 * (nnz_a + n_h + 1) + 12 * nnz_h


def cpu_sample(bundle, x, budget_s=3.0):
    """Oracle port (reference algorithm) on a contiguous row slab; returns
    (GB/s, seconds, rows, bytes)."""
    import oracle

    cp = bundle.triple.matrices[: bundle.n_terms]
    n_h, n_xi = x.shape
    rows = max(256, n_h // 64)
    t0 = time.perf_counter()
    oracle.kron_apply_rows(cp, bundle.stiffness, x, (0, rows))
    dt = time.perf_counter() - t0
    rows = int(min(n_h, max(rows, rows * budget_s / max(dt, 1e-3))))
    r0 = (n_h - rows) // 2
    a = bundle.stiffness[0][r0:r0 + rows]
    touched = np.unique(a.indices).size
    nnz = a.nnz
    nnz_h = sum(int(h.nnz) for h in cp)
    b = 8 * n_xi * (touched + rows) + 8 * bundle.n_terms * nnz + 4 * (nnz + rows + 1) + 12 * nnz_h
    t0 = time.perf_counter()
    oracle.kron_apply_rows(cp, bundle.stiffness, x, (r0, r0 + rows))
    dt = time.perf_counter() - t0
    return b / dt / 1e9, dt, rows, b


def reduce_max(value: float, device=None) -> float:
    """Max over ranks (the contract's "max over ranks" timing); identity when
    not distributed.  NCCL on the GPU path, gloo in the CPU tests."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_gbs(bytes_per_step: int, steps: int, world: int, seconds_max: float) -> float:
    """Weak scaling: every rank runs its own `steps` matvecs; the job's
    throughput is all ranks' bytes over the slowest rank's time."""
    return world * steps * bytes_per_step / seconds_max / 1e9


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    ws, rank, _ = _dist()
    if ws > 1 and rank != 0:
        return
    from paper_2512_23804_b200.problems import build_problem

    bundle = build_problem(4)
    x = np.random.default_rng(SEED).standard_normal((bundle.n_h, bundle.n_xi))
    vals = []
    for i in range(args.warmup + args.steps):
        gbs, dt, rows, b = cpu_sample(bundle, x, budget_s=args.ref_budget)
        if i >= args.warmup:
            vals.append((gbs, dt, rows, b))
    value = statistics.median(v[0] for v in vals)
    rows = vals[-1][2]
    line = {
        "impl": "reference",
        "metric": "galerkin_matvec_gbs",
        "value": value,
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(v[1] for v in vals),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded N(0,1) V, BASELINE cfg4 operators)",
        "config": {"workload": "cfg4 Galerkin matvec, row sample", "n_h": bundle.n_h, "n_xi": bundle.n_xi,
                   "n_t": bundle.n_terms, "sample_rows": rows},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "port",
                         "sample": f"rows [{(bundle.n_h - rows) // 2}, +{rows}) of the cfg4 matvec per step; "
                                   "NumPy/SciPy restatement of sgkkt kron_apply (scipy sparsetools holds the GIL: 1 core)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_solve:
        line["solves"] = {"cfg2": cpu_solve_block(2, 1e-2)}
        if not args.no_solve_cfg5:
            # the headline control solve on the host ("the full CPU
            # FGMRES solve"): hGSoc inside the reference FGMRES, beta = 1e-2
            line["solves"]["cfg5"] = cpu_solve_block(5, 1e-2, minres=False)
    print(json.dumps(line), flush=True)


def cpu_solve_block(cfg_id, beta, minres=True):
    """Time-to-solution of the oracle port (reference algorithms: hGSoc inside
    the reference FGMRES; block-diagonal hGS preconditioned MINRES) on the host."""
    import scipy.sparse as sp

    import oracle
    from paper_2512_23804_b200.problems import build_problem, steady_system

    b = build_problem(cfg_id, beta=beta)
    s = steady_system(b)
    n_h, n_xi = s.n_h, s.n_xi
    size = n_h * n_xi
    cp = s.triple.matrices[: s.n_terms]
    w = s.triple.weight_diagonal
    unpack = lambda v: [v[i * size:(i + 1) * size].reshape(n_h, n_xi) for i in range(3)]
    pack = lambda blocks: np.concatenate([np.asarray(x).ravel() for x in blocks])
    op = lambda v: pack(oracle.steady_kkt_apply(s.mass, s.stiffness, cp, w, s.beta, *unpack(v)))
    rhs = np.zeros(3 * size)
    rhs[:size] = np.asarray(s.mass @ s.target).ravel()
    out = {}
    t0 = time.perf_counter()
    m, a0 = s.mass, s.stiffness[0]
    kkt_lu = oracle.splu_ref(sp.bmat([[m, None, -a0], [None, s.beta * m, m], [-a0, m, None]], format="csr"))
    t_setup = time.perf_counter() - t0
    soc = lambda v: pack(oracle.coupled_sweep_apply(m, s.stiffness, s.triple.matrices, s.triple.objective_weight,
                                                    s.beta, b.partition.boundaries, s.n_terms, kkt_lu, *unpack(v)))
    t0 = time.perf_counter()
    x, its, conv, _ = oracle.fgmres(op, soc, rhs, 1e-8)
    out["hgsoc_fgmres"] = {"iterations": its, "converged": bool(conv), "seconds": time.perf_counter() - t0,
                           "setup_seconds": t_setup}
    if not minres:
        return {f"beta={beta:g}": out, "cores": 1}
    t0 = time.perf_counter()
    lead = oracle.splu_ref(oracle.shifted_lead(m, s.stiffness, s.beta, s.gamma)[0])
    t_setup = time.perf_counter() - t0
    bd = lambda v: pack(oracle.steady_precond_apply(m, s.stiffness, cp, w, s.beta, s.gamma, b.partition.boundaries,
                                                    s.n_terms, lead, *unpack(v)))
    t0 = time.perf_counter()
    x, its, conv, _ = oracle.minres(op, bd, rhs, 1e-8)
    out["blockdiag_hgs_minres"] = {"iterations": its, "converged": bool(conv), "seconds": time.perf_counter() - t0,
                                   "setup_seconds": t_setup}
    return {f"beta={beta:g}": out, "cores": 1}


# time-to-solution of the reference itself (`sgkkt` fgmres + CoupledSweepPreconditioner
# / SteadyKKTPreconditioner + oracle MINRES) on the full config-5 inputs, one core of
# the BUILD container (tests/golden/make_solves.py; fixtures tests/golden/solves/)
REF_CFG5_SECONDS = {
    "beta=0.01": {"hgsoc_fgmres": {"iterations": 7, "seconds": 180.5},
                  "blockdiag_hgs_minres": {"iterations": 37, "seconds": 702.3}},
    "beta=0.0001": {"hgsoc_fgmres": {"iterations": 11, "seconds": 281.3},
                    "blockdiag_hgs_minres": {"iterations": 36, "seconds": 684.3}},
    "beta=1e-06": {"hgsoc_fgmres": {"iterations": 10, "seconds": 270.1},
                   "blockdiag_hgs_minres": {"iterations": 32, "seconds": 615.3}},
}


def cpu_iteration_sample(cfg_id, beta):
    """Bounded CPU sample of the config-5 solve on this host (oracle port, 1
    core): one hGSoc apply (LU factor excluded, timed separately) and one KKT
    matvec = the cost of one FGMRES iteration; projected to the reference's
    iteration count.  The full solves of the reference itself are in
    REF_CFG5_SECONDS (build container) and the reference arm times the
    beta = 1e-2 solve end to end on this host."""
    import scipy.sparse as sp

    import oracle
    from paper_2512_23804_b200.problems import build_problem, steady_system

    b = build_problem(cfg_id, beta=beta)
    s = steady_system(b)
    n_h, n_xi = s.n_h, s.n_xi
    cp = s.triple.matrices[: s.n_terms]
    rng = np.random.default_rng(SEED)
    blocks = [rng.standard_normal((n_h, n_xi)) for _ in range(3)]
    m, a0 = s.mass, s.stiffness[0]
    t0 = time.perf_counter()
    kkt_lu = oracle.splu_ref(sp.bmat([[m, None, -a0], [None, s.beta * m, m], [-a0, m, None]], format="csr"))
    t_fac = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.coupled_sweep_apply(m, s.stiffness, s.triple.matrices, s.triple.objective_weight, s.beta,
                               b.partition.boundaries, s.n_terms, kkt_lu, *blocks)
    t_apply = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.steady_kkt_apply(m, s.stiffness, cp, s.triple.weight_diagonal, s.beta, *blocks)
    t_mv = time.perf_counter() - t0
    its = REF_CFG5_SECONDS[f"beta={beta:g}"]["hgsoc_fgmres"]["iterations"]
    return {f"beta={beta:g}": {"hgsoc_apply_s": t_apply, "kkt_matvec_s": t_mv, "lu_factor_s": t_fac,
                               "projected_hgsoc_fgmres_s": its * (t_apply + t_mv), "iterations": its,
                               "cores": 1, "kind": "port",
                               "reference_sgkkt_build_container": REF_CFG5_SECONDS}}


def _event_time(fn, steps, stream):
    import torch

    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(steps):
        fn()
    end.record(stream)
    end.synchronize()
    return start.elapsed_time(end) / 1e3


def solve_block(cfg_id, betas, with_cpu=False, lead_solvers=("lu", "lu_nd", "lu_tp", "fastdiag")):
    """Time-to-solution of the control configs on the GPU (setup reported
    separately).  Lead solvers: "lu" = the reference's SuperLU factors replayed
    by the GPU triangular solves (the reference algorithm); "fastdiag" = the
    depth-free Kronecker-sum solve, keys suffixed
    "[fastdiag]"."""
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, fgmres, minres
    from paper_2512_23804_b200.operators import steady_kkt_apply_device
    from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, build_steady_preconditioner
    from paper_2512_23804_b200.problems import build_problem, steady_system

    out = {}
    t0 = time.perf_counter()
    bundle = build_problem(cfg_id)
    t_asm = time.perf_counter() - t0
    for beta in betas:
        sys_ = steady_system(bundle, beta=beta)
        n = sys_.block_size()
        shape = (sys_.n_h, sys_.n_xi)
        rhs = np.zeros(3 * n)
        rhs[:n] = np.asarray(sys_.mass @ sys_.target).ravel()
        b = torch.as_tensor(rhs).cuda()

        def split(v):
            return [v[i * n:(i + 1) * n].view(shape) for i in range(3)]

        def op(v):
            o = torch.empty_like(v)
            steady_kkt_apply_device(sys_, *split(v), tuple(split(o)))
            return o

        rec = {}
        variants = []
        for ls in lead_solvers:
            sfx = "" if ls == "lu" else f"[{ls}]"
            if ls != "lu_nd":  # P~ is indefinite and keeps COLAMD under lu_nd: same as "lu"
                variants.append((f"hgsoc_fgmres{sfx}",
                                 lambda ls=ls: build_coupled_preconditioner(sys_, bundle.partition, lead_solver=ls),
                                 fgmres))
            if ls == "lu_tp":  # the SPD lead does not pivot: same factors as "lu"
                continue
            variants.append((f"blockdiag_hgs_minres{sfx}",
                             lambda ls=ls: build_steady_preconditioner(sys_, bundle.partition, "cheb5", lead_solver=ls),
                             minres))
        for name, builder, solver in variants:
            t0 = time.perf_counter()
            prec = builder()
            # first apply compiles programs and uploads factors (setup)
            warm = torch.zeros(3 * n, dtype=torch.float64, device="cuda")
            warm[0] = 1.0
            prec.apply_device(*split(warm), outs=tuple(split(torch.empty_like(warm))))
            torch.cuda.synchronize()
            t_setup = time.perf_counter() - t0

            def pr(v, prec=prec):
                o = torch.empty_like(v)
                prec.apply_device(*split(v), outs=tuple(split(o)))
                return o

            times = []
            for _ in range(2):  # first solve (cold allocator) and a warm repeat
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                x, rep = solver(op, pr, b, FgmresConfig(tol=1e-8, max_iters=500))
                torch.cuda.synchronize()
                times.append(time.perf_counter() - t0)
            r = op(x)
            true_res = float(torch.linalg.vector_norm(b - r) / torch.linalg.vector_norm(b))
            rec[name] = {"iterations": rep.iterations, "converged": bool(rep.converged),
                         "seconds": times[1], "first_solve_seconds": times[0], "setup_seconds": t_setup,
                         "true_rel_residual": true_res, "tol": 1e-8}
        out[f"beta={beta:g}"] = rec
    out["assembly_seconds"] = t_asm
    return out


def forward_block(cfg_id, n_taus=None, lead_solvers=("lu", "fastdiag")):
    """BASELINE configs 1 and 3 (forward problem -div(a grad u) = 1): one
    Galerkin matvec (GB/s, kernel path) and hGS-CG to 1e-8 per truncation
    n_tau and lead solver (setup separate)."""
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, cg
    from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply
    from paper_2512_23804_b200.preconditioners import build_sweep
    from paper_2512_23804_b200.problems import build_problem

    t0 = time.perf_counter()
    b = build_problem(cfg_id)
    t_asm = time.perf_counter() - t0
    cp = b.triple.matrices[: b.n_terms]
    shape = (b.n_h, b.n_xi)
    op = KroneckerSumOperator(couplings=cp, operators=b.stiffness)
    x = torch.as_tensor(np.random.default_rng(SEED).standard_normal(shape)).cuda()
    stream = torch.cuda.current_stream()
    kron_apply(op, x)
    torch.cuda.synchronize()
    t_mv = _event_time(lambda: kron_apply(op, x), 10, stream) / 10
    out = {"n_h": b.n_h, "n_xi": b.n_xi, "n_t": b.n_terms, "assembly_seconds": t_asm,
           "matvec_ms": t_mv * 1e3, "matvec_gbs": op.algorithmic_bytes() / t_mv / 1e9,
           "matvec_kernel": op.program([(0, b.n_xi)], (0, b.n_xi), 0, op.n_terms).host.stats.get("mode", "program")}
    rhs = torch.as_tensor(b.forward_rhs().ravel()).cuda()
    for n_tau in (n_taus or [b.n_terms]):
        for ls in lead_solvers:
            t0 = time.perf_counter()
            _, sweep = build_sweep(cp, b.stiffness, b.partition, n_tau, lead_solver=ls, mass=b.mass)
            sweep.apply_device(x)
            torch.cuda.synchronize()
            t_setup = time.perf_counter() - t0
            apply_op = lambda v: kron_apply(op, v.view(shape)).reshape(-1)
            apply_pr = lambda v, sw=sweep: sw.apply_device(v.view(shape)).reshape(-1)
            times = []
            for _ in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                xs, rep = cg(apply_op, apply_pr, rhs, FgmresConfig(tol=1e-8))
                torch.cuda.synchronize()
                times.append(time.perf_counter() - t0)
            res = float(torch.linalg.vector_norm(rhs - apply_op(xs)) / torch.linalg.vector_norm(rhs))
            sfx = "" if ls == "lu" else f"[{ls}]"
            out[f"hgs_cg{sfx} n_tau={n_tau}"] = {"iterations": rep.iterations, "converged": bool(rep.converged),
                                                "seconds": times[1], "first_solve_seconds": times[0],
                                                "setup_seconds": t_setup, "true_rel_residual": res, "tol": 1e-8}
    return out


def apply_breakdown(cfg_id, beta=1e-2):
    """one KKT matvec (GB/s vs the HBM floor) and one hGSoc apply
    split into its coupling launches and P~ solves, LU and fastdiag leads
    (CUDA events, warm, 5 repetitions each)."""
    import torch

    from paper_2512_23804_b200.device import run_program
    from paper_2512_23804_b200.operators import steady_kkt_apply_device
    from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner
    from paper_2512_23804_b200.problems import build_problem, steady_system

    stream = torch.cuda.current_stream()

    def ms(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        return _event_time(fn, reps, stream) / reps * 1e3

    b = build_problem(cfg_id)
    s = steady_system(b, beta=beta)
    shape = (s.n_h, s.n_xi)
    rng = np.random.default_rng(SEED)
    blocks = [torch.as_tensor(rng.standard_normal(shape)).cuda() for _ in range(3)]
    outs = tuple(torch.empty_like(blocks[0]) for _ in range(3))
    t_kkt = ms(lambda: steady_kkt_apply_device(s, *blocks, outs))
    peak, _ = _peaks()
    out = {"beta": beta, "kkt_matvec_ms": t_kkt, "kkt_algorithmic_bytes": s.algorithmic_bytes(),
           "kkt_gbs": s.algorithmic_bytes() / (t_kkt * 1e-3) / 1e9}
    out["kkt_hbm_frac"] = out["kkt_gbs"] / peak
    for ls in ("lu", "fastdiag"):
        soc = build_coupled_preconditioner(s, b.partition, lead_solver=ls)
        fac = soc.kkt_factor.device_factors
        fwd, bwd = soc._programs()
        ranges = b.partition.ranges()
        levels = list(zip(ranges, fwd)) + list(zip(reversed(ranges[:-1]), bwd))
        rec = {"apply_ms": ms(lambda: soc.apply_device(*blocks, outs=outs)), "levels": []}
        for (lo, hi), prog in levels:
            segs = [(o, lo) for o in outs]
            tc = ms(lambda: run_program(s.pattern, prog, [(o, 0) for o in outs], segs, [(r, lo) for r in blocks],
                                        alpha=[1.0] * 3, beta=[1.0] * 3))
            ts = ms(lambda: fac.solve_segments(segs, segs, hi - lo))
            rec["levels"].append({"width": hi - lo, "coupling_ms": tc, "solve_ms": ts})
        rec["couplings_ms"] = sum(lv["coupling_ms"] for lv in rec["levels"])
        rec["solves_ms"] = sum(lv["solve_ms"] for lv in rec["levels"])
        out[f"hgsoc_{ls}"] = rec
    return out


def time_solve_block(with_cpu: bool):
    """all-at-once time-dependent KKT with the PINT
    preconditioner inside the reference FGMRES (tol 1e-6, Chebyshev-5, hGS
    Richardson-1, n_tau = n_A) on the paper's (3,3) lognormal setting:
    n=32 (N=961), m=3, p=3 (n_xi=20), coefficient degree 6 (84 terms), N_t=8."""
    import torch

    from paper_2512_23804_b200.krylov import FgmresConfig, fgmres
    from paper_2512_23804_b200.problems import ConfigSpec, build_problem, steady_system
    from paper_2512_23804_b200.timedep import (TimeKKT, build_time_preconditioner, build_time_stencil,
                                               time_kkt_apply, time_rhs, to_device_layout)

    spec = ConfigSpec("time_paper", "control", 32, 3, 3, "hermite", "lognormal", 0.2, 1.0,
                      coefficient_degree=6, beta=1e-4, lo=-1.0, hi=1.0)
    b = build_problem(spec, kl_method="dense")
    st = steady_system(b)
    sys_ = TimeKKT(steady=st, stencil=build_time_stencil(8), initial_state=np.zeros((st.n_h, st.n_xi)))
    rhs = time_rhs(sys_)
    bd = to_device_layout(sys_, rhs)
    out = {"dofs": 3 * sys_.block_size(), "n_t": 8, "n_xi": st.n_xi, "n_terms": st.n_terms}
    for ls in ("lu", "fastdiag"):
        t0 = time.perf_counter()
        prec = build_time_preconditioner(sys_, b.partition, "cheb5", lead_solver=ls)
        prec.apply(bd)
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t0
        times = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, rep = fgmres(lambda v: time_kkt_apply(sys_, v), lambda v: prec.apply(v), bd, FgmresConfig(tol=1e-6))
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        out["gpu" if ls == "lu" else f"gpu[{ls}]"] = {
            "iterations": rep.iterations, "converged": bool(rep.converged), "seconds": times[1],
            "first_solve_seconds": times[0], "setup_seconds": t_setup}
    if with_cpu:
        import oracle

        m, a = st.mass, st.stiffness
        cp = st.triple.matrices[: st.n_terms]
        lead = oracle.splu_ref(oracle.time_lead(m, a, st.beta, st.gamma, 8)[0])
        op = lambda v: oracle.time_kkt_apply(m, a, cp, st.triple.weight_diagonal, st.beta, 8, v)
        pr = lambda v: oracle.time_precond_apply(m, a, cp, st.triple.weight_diagonal, st.beta, st.gamma,
                                                 b.partition.boundaries, st.n_terms, lead, 8, v)
        t0 = time.perf_counter()
        _, its, conv, _ = oracle.fgmres(op, pr, rhs, 1e-6)
        out["cpu_port"] = {"iterations": its, "converged": bool(conv), "seconds": time.perf_counter() - t0, "cores": 1}
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2512_23804_b200 import _lib
    from paper_2512_23804_b200.operators import kron_apply
    from paper_2512_23804_b200.preconditioners import build_sweep
    from paper_2512_23804_b200.problems import build_problem

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    bundle = build_problem(4)
    cp = bundle.triple.matrices[: bundle.n_terms]
    from paper_2512_23804_b200.operators import KroneckerSumOperator

    op = KroneckerSumOperator(couplings=cp, operators=bundle.stiffness)
    rng = np.random.default_rng(SEED + rank)
    x_host = rng.standard_normal((bundle.n_h, bundle.n_xi))
    x = torch.as_tensor(x_host).to(dev)
    w = torch.empty_like(x)
    nnz_h = sum(int(h.nnz) for h in cp)
    B = matvec_bytes(bundle.n_h, bundle.n_xi, bundle.n_terms, bundle.stiffness[0].nnz, nnz_h)
    assert B == op.algorithmic_bytes()
    from paper_2512_23804_b200.device import run_program

    prog = op.program([(0, bundle.n_xi)], (0, bundle.n_xi), 0, op.n_terms)
    stream = torch.cuda.current_stream()

    def step():
        run_program(op.pattern, prog, [(x, 0)], [(w, 0)], alpha=[1.0], beta=[0.0])

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # correctness spot-check on a row slab against the oracle (outside the timed region)
    import oracle

    r0 = bundle.n_h // 2
    ref = oracle.kron_apply_rows(cp, bundle.stiffness, x_host, (r0, r0 + 64))
    got = w[r0:r0 + 64].cpu().numpy()
    spot_err = float(np.abs(got - ref).max() / np.abs(ref).max())

    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        t = _event_time(step, args.steps, stream)
    launches = _lib.launch_count() - l0
    torch.cuda.synchronize()
    t = reduce_max(t, dev)
    if ws > 1:
        dist.barrier()
    value = whole_job_gbs(B, args.steps, ws, t)
    kernel_avg = t / args.steps
    # per-matvec distribution (median and best), separate pass
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for i in range(args.steps):
        step()
        evs[i + 1].record(stream)
    evs[-1].synchronize()
    per = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)])
    per_step = {"median_ms": float(np.median(per)), "best_ms": float(per.min()), "worst_ms": float(per.max()),
                "median_gbs": B / (float(np.median(per)) * 1e-3) / 1e9, "best_gbs": B / (float(per.min()) * 1e-3) / 1e9}

    # e2e through the public API with pinned host buffers
    xp = torch.from_numpy(x_host).pin_memory()
    wp = torch.empty_like(xp).pin_memory()
    for _ in range(2):
        kron_apply(op, xp, out=wp)
    torch.cuda.synchronize()
    e2e_steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(e2e_steps):
        kron_apply(op, xp, out=wp)
    ev1.record(stream)
    ev1.synchronize()
    t_e2e = ev0.elapsed_time(ev1) / 1e3
    e2e_err = float(np.abs(wp.numpy() - w.cpu().numpy()).max())
    t_e2e = reduce_max(t_e2e, dev)
    e2e_value = whole_job_gbs(B, e2e_steps, ws, t_e2e)
    # the PCIe roofline of the e2e path on this box: both directions of the
    # step's copies running concurrently (raw copies, no kernel)
    yd = torch.empty_like(x)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def duplex():
        with torch.cuda.stream(s1):
            x.copy_(xp, non_blocking=True)
        with torch.cuda.stream(s2):
            wp.copy_(yd, non_blocking=True)
        stream.wait_stream(s1)
        stream.wait_stream(s2)

    duplex()
    torch.cuda.synchronize()
    t_dup = _event_time(duplex, 3, stream) / 3
    pcie = {"duplex_copy_ms": t_dup * 1e3, "duplex_gbs": 2 * xp.numel() * 8 / t_dup / 1e9,
            "frac_of_duplex_copy_time": t_dup / (t_e2e / e2e_steps)}

    peak, peak_kind = _peaks()
    achieved = B / kernel_avg / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get("matvec_kernel_cfg4_bytes")
        except Exception:
            traffic = None
    line = {
        "metric": "galerkin_matvec_gbs",
        "value": value,
        "unit": "GB/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * kernel_avg,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded N(0,1) V; BASELINE cfg4 operators: Q1 256x256 unit square, affine KL, Legendre m=10 p=4)",
        "config": {"workload": "cfg4 Galerkin matvec W = sum_t A_t V H_t", "n_h": bundle.n_h, "n_xi": bundle.n_xi,
                   "n_t": bundle.n_terms, "nnz_A": int(bundle.stiffness[0].nnz), "nnz_H": nnz_h,
                   "algorithmic_bytes": B, "l2": "inputs larger than L2 (V 520.7 MB, W 520.7 MB per step)",
                   "parallelism": f"replica x{ws} (independent matvecs per GPU)",
                   "spot_check_rel_err_vs_oracle": spot_err},
        "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": int(x.numel() * 8),
                "d2h_bytes_per_step": int(w.numel() * 8), "api": "kron_apply(op, pinned CPU tensor, out=pinned)",
                "max_abs_diff_vs_device": e2e_err, "pcie_roofline": pcie},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": (((("stencil9_grid_kernel<TMA> (grid form, sliding V window, TMA/mbarrier pipeline"
                                   if os.environ.get("SGKKT_GRID9", "1") == "1" and os.environ.get("SGKKT_GRID_TMA") != "0"
                                   else "stencil9_tma_kernel (TMA/mbarrier pipeline" if os.environ.get("SGKKT_S9_TMA") != "0"
                                   else "stencil9_ws_kernel (named barriers") + ": 8 producer + 8 consumer warps)")
                                 if 6 <= prog.host.stats.get("n_groups", 0) <= 8 and os.environ.get("SGKKT_S9_WS") != "0"
                                 else "stencil9_kernel")
                                if prog.host.stats.get("mode") == "stencil9" else "program_kernel")
                     + " (cfg4 full matvec)", "fp64_flops_per_launch": None},
        "clocks": clk.summary(),
    }
    prog_stats = prog.host.stats
    line["config"]["schedule"] = prog_stats
    line["per_step"] = per_step
    # fp64 work actually issued per launch (the kernel is DFMA-heavy: SURVEY §7 H1)
    useful = 2 * bundle.stiffness[0].nnz * prog_stats["n_products"] + 2 * bundle.n_h * prog_stats["n_gather"]
    line["roofline"]["fp64_flops_per_launch"] = useful
    line["roofline"]["fp64_tflops"] = useful / kernel_avg / 1e12
    line["roofline"]["fp64_peak_tflops"] = FP64_PEAK_TFLOPS
    line["roofline"]["fp64_frac"] = useful / kernel_avg / 1e12 / FP64_PEAK_TFLOPS
    if rank == 0 and not args.no_cpu:
        gbs, dt, rows, b = cpu_sample(bundle, x_host, budget_s=args.ref_budget)
        line["cpu_baseline"] = {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "port",
                                "sample": f"{rows} contiguous output rows of the cfg4 matvec ({b / 1e6:.1f} MB algorithmic, "
                                          f"{dt:.2f} s); NumPy/SciPy oracle port of sgkkt kron_apply, 1 core (GIL-bound)"}
        if not args.no_solve and not args.no_solve_cfg5:
            line["cpu_baseline"]["solves"] = {"cfg5": cpu_iteration_sample(5, 1e-2)}
    if rank == 0 and not args.no_solve:
        solves = {"cfg2": solve_block(2, [1e-2])}
        solves["cfg1_forward"] = forward_block(1)
        solves["cfg3_forward"] = forward_block(3, [1, 7, 924])
        if not args.no_solve_cfg5:
            solves["cfg5"] = solve_block(5, [1e-2, 1e-4, 1e-6])
            solves["cfg5_apply_breakdown"] = apply_breakdown(5)
        if not args.no_solve_time:
            solves["time_dependent"] = time_solve_block(args.time_cpu)
        line["solves"] = solves
    if rank == 0 and args.table_out:
        from paper_2512_23804_b200.problems import build_problem
        from paper_2512_23804_b200.tables import emit_table, experiment_rows

        rows = experiment_rows(build_problem(2), lead_solver=args.table_lead)
        b5 = build_problem(5)
        for beta in (1e-2, 1e-4, 1e-6):
            rows += experiment_rows(b5, n_taus=[b5.n_terms], beta=beta, lead_solver=args.table_lead)
        with open(args.table_out, "w") as fh:
            fh.write(emit_table(rows, "markdown" if args.table_out.endswith(".md") else "csv"))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--solve-cfg5", action="store_true", help="(default on; kept for compatibility)")
    ap.add_argument("--no-solve-cfg5", action="store_true", help="skip the cfg5 beta sweep")
    ap.add_argument("--solve-time", action="store_true", help="(default on; kept for compatibility)")
    ap.add_argument("--no-solve-time", action="store_true", help="skip the time-dependent PINT solve (SURVEY 8(f) row 1)")
    ap.add_argument("--time-cpu", action="store_true", help="also time the CPU port of the time-dependent solve")
    ap.add_argument("--ref-budget", type=float, default=3.0)
    ap.add_argument("--table-out", default=None,
                    help="also write the reference-schema result table (.csv or .md) of the cfg2/cfg5 experiment rows")
    ap.add_argument("--table-lead", choices=["lu", "fastdiag"], default="lu")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
