"""Critical-path timing of the grouped triangular solve (debug build with
-DSGK_TRI_TRACE into paper_2512_23804_b200/libsgkkt_tritrace.so):
python tools/tri_trace.py cfg level"""
import ctypes, os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
os.environ.setdefault("SGKKT_B200_LIB", str(ROOT / "paper_2512_23804_b200" / "libsgkkt_tritrace.so"))
sys.path.insert(0, str(ROOT))
import numpy as np, torch
from paper_2512_23804_b200 import _lib
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
lvl = int(sys.argv[2]) if len(sys.argv) > 2 else 0
b = build_problem(cfg); s = steady_system(b)
fac = build_coupled_preconditioner(s, b.partition).kkt_factor.device_factors
lo, hi = b.partition.ranges()[lvl]
blk = [torch.randn((s.n_h, s.n_xi), dtype=torch.float64, device="cuda") for _ in range(3)]
out = [torch.empty_like(blk[0]) for _ in range(3)]
for _ in range(3):
    fac.solve_segments([(t, lo) for t in blk], [(t, lo) for t in out], hi - lo)
torch.cuda.synchronize()
lib = _lib.lib()
bad = (ctypes.c_int * 2)()
lib.sgk_tri_bad_read(bad)
print("tasks that passed the dependency wait with an unset flag (fwd, bwd):", bad[0], bad[1])
for fwd, bufs, gs in ((1, fac.gl_bufs, fac.gl), (0, fac.gu_bufs, fac.gu)):
    ng = gs.n_groups
    width = hi - lo
    cw = 1 if width <= 8 else (2 if width <= 40 else 4)
    nch = -(-width // cw)
    nt = ng * nch
    arr = (ctypes.c_ulonglong * (8 * nt))()
    lib.sgk_tri_trace_read(arr, fwd, nt)
    tr = np.frombuffer(arr, dtype=np.uint64).reshape(nt, 8)[:, :7].astype(np.float64)
    order = bufs[4].cpu().numpy()
    dptr = bufs[10].cpu().numpy(); deps = bufs[11].cpu().numpy()
    t0 = tr[:, 0].min()
    c5 = c6 = c7 = 0.0
    tr -= t0
    pos = np.empty(ng, np.int64); pos[order] = np.arange(ng)  # ticket of group (chunk 0)
    done = tr[:, 4]
    # chunk 0 only
    notif, comp, ph1, ph2, ph3, wait = [], [], [], [], [], []
    for tk in range(0, nt, nch):
        g = order[tk // nch]
        ds = deps[dptr[g]:dptr[g + 1]]
        last = max((done[pos[d] * nch] for d in ds), default=tr[tk, 0])
        notif.append(tr[tk, 1] - max(last, tr[tk, 0]))
        wait.append(tr[tk, 1] - tr[tk, 0])
        ph1.append(tr[tk, 2] - tr[tk, 1]); ph2.append(tr[tk, 3] - tr[tk, 2]); ph3.append(tr[tk, 4] - tr[tk, 3])
    f = lambda a: f"{np.median(a)/1e3:.2f}/{np.mean(a)/1e3:.2f}"
    print(f"{'L' if fwd else 'U'} width {width} groups {ng} tasks {nt} total {done.max()/1e3:.0f} us; median/mean us: "
          f"notify {f(notif)} phase1 {f(ph1)} chain {f(ph2)} [setup {c5/1e3:.2f} loop {c6/1e3:.2f} sync {c7/1e3:.2f}] write+fence {f(ph3)} wait {f(wait)}")
    if fwd and nch == 1:
        rp = bufs[0].cpu().numpy(); sp_ = bufs[9].cpu().numpy(); gp = bufs[3].cpu().numpy()
        ph1a = np.array(ph1)
        top = np.argsort(-ph1a)[:12]
        print("  top phase-1 tasks (ticket, rows, outside entries, phase1 us, done us):")
        for tk in top:
            g = order[tk]
            a, b_ = gp[g], gp[g + 1]
            ne = int((sp_[a:b_] - rp[a:b_]).sum())
            print(f"   {tk:5d} rows {b_ - a:2d} entries {ne:7d} phase1 {ph1a[tk]/1e3:8.1f} done {done[tk]/1e3:8.1f}")
        # critical path walk back from the last task
        cp, tk = [], int(np.argmax(done))
        while True:
            g = order[tk]; cp.append(tk)
            ds = deps[dptr[g]:dptr[g + 1]]
            if not len(ds): break
            tk = int(max((pos[d] for d in ds), key=lambda q: done[q]))
        cp = cp[::-1]
        tot1 = sum(ph1a[q] for q in cp)
        print(f"  critical path: {len(cp)} tasks, sum phase1 {tot1/1e3:.0f} us, end {done.max()/1e3:.0f} us")
        for tk in (4377, 4376, 4375):
            if tk >= nt: continue
            g = order[tk]; ds = deps[dptr[g]:dptr[g + 1]]
            dd = sorted(((done[pos[d]], pos[d]) for d in ds), reverse=True)[:3]
            print(f"  task {tk} group {g}: t0..t4 {[round(x/1e3,1) for x in tr[tk,:5]]} n_deps {len(ds)} latest deps (done, ticket) {[(round(a/1e3,1), int(b)) for a, b in dd]}")
    fin = np.sort(done)
    q = [fin[int(f * (len(fin) - 1))] / 1e3 for f in (0.5, 0.9, 0.99, 1.0)]
    grp_done = np.array([done[pos[g] * nch:(pos[g] + 1) * nch].max() for g in range(ng)])
    last = np.argsort(grp_done)[-40:]
    print(f"  task completion quantiles (us): 50% {q[0]:.0f}  90% {q[1]:.0f}  99% {q[2]:.0f}  100% {q[3]:.0f};"
          f" last 40 groups finish between {grp_done[last].min()/1e3:.0f} and {grp_done.max()/1e3:.0f} us")
