"""Critical-path anatomy of the wide triangular solve (trace build:
`make trace` -> build_variants/libsgkkt_triwtrace.so):
python tools/triw_trace.py width
Per task (tile, chunk) the kernel stamps: 0 ticket, 1 dependencies ready,
2 segments done, 3 counter done (multi-tile groups), 4 flag published
(finaliser only; else = 0), 5 end.  Prints per-phase medians and the
per-group-level timeline."""
import ctypes, os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
os.environ.setdefault("SGKKT_B200_LIB", str(ROOT / "build_variants" / "libsgkkt_triwtrace.so"))
sys.path.insert(0, str(ROOT))
import numpy as np, torch
from paper_2512_23804_b200 import _lib
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system
width = int(sys.argv[1]) if len(sys.argv) > 1 else 64
b = build_problem(5); s = steady_system(b)
fac = build_coupled_preconditioner(s, b.partition).kkt_factor.device_factors
blk = [torch.randn((s.n_h, width), dtype=torch.float64, device="cuda") for _ in range(3)]
out = [torch.empty_like(blk[0]) for _ in range(3)]
for _ in range(3):
    fac.solve_segments([(t, 0) for t in blk], [(t, 0) for t in out], width)
torch.cuda.synchronize()
lib = _lib.lib()
lib.sgk_triw_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
ch = int(lib.sgk_trisolve_wide_chunk_cols(width))
nch = -(-width // ch)
for fwd, tw, bufs in ((1, fac.wl, fac.wl_bufs), (0, fac.wu, fac.wu_bufs)):
    nt = tw.n_tiles * nch
    arr = np.zeros((nt, 6), np.uint64)
    lib.sgk_triw_trace_read(arr.ctypes.data, fwd, nt)
    tr = arr.astype(np.float64)
    tr -= tr[:, 0].min()
    tr /= 1e3  # us
    tile_group = bufs[0].cpu().numpy()
    tile = np.arange(nt) // nch
    g = tile_group[tile]
    fin = tr[:, 4] > 0
    span = tr[:, 5].max()
    print(f"{'L' if fwd else 'U'}: tasks {nt}, span {span:.0f} us, finalisers {fin.sum()}")
    print(f"   median us: wait {np.median(tr[:, 1] - tr[:, 0]):.2f}  segments {np.median(tr[:, 2] - tr[:, 1]):.2f}"
          f"  counter {np.median(tr[fin, 3] - tr[fin, 2]) if fin.any() else 0:.2f}"
          f"  finalise {np.median(tr[fin, 4] - tr[fin, 3]) if fin.any() else 0:.2f}")
    # group finish times in topological order
    gf = {}
    for i in np.nonzero(fin)[0]:
        gf[int(g[i])] = max(gf.get(int(g[i]), 0.0), tr[i, 4])
    order = []
    for i in range(nt):
        if int(g[i]) not in order[-1:]:
            order.append(int(g[i]))
    fins = np.array([gf.get(x, np.nan) for x in order])
    q = np.linspace(0, len(fins) - 1, 11).astype(int)
    print("   group finish (us) at deciles of the topological order:", np.round(fins[q], 0))
    # time from deps ready to segments done, per tile size (entries)
    e0 = bufs[6].cpu().numpy(); e1 = bufs[7].cpu().numpy(); ts = bufs[1].cpu().numpy()
    cs = np.concatenate([[0], np.cumsum(e1 - e0)])
    ent = (cs[ts[1:]] - cs[ts[:-1]])[tile]
    for lo, hi in ((0, 128), (128, 512), (512, 1025)):
        sel = (ent >= lo) & (ent < hi)
        if sel.any():
            print(f"   tiles with {lo}-{hi} entries: {sel.sum()}, segments phase median {np.median(tr[sel, 2] - tr[sel, 1]):.2f} us")

    # dense-region chain: per block, publish(i-1) -> detect(i) -> applied -> publish(i)
    kind = bufs[12].cpu().numpy()
    dk = np.nonzero(kind[tile] == 1)[0]
    if len(dk):
        c0 = dk[(np.arange(nt)[dk] % nch) == 0]  # chunk 0 of each dense task
        pub = tr[c0, 4]
        det = tr[c0, 1]
        app = tr[c0, 2]
        if len(c0) > 2:
            prop = det[1:] - pub[:-1]
            print(f"   dense chain ({len(c0)} blocks, chunk 0): median us: publish(i-1)->detect(i) {np.median(prop):.2f}"
                  f"  detect->applied {np.median(app[1:] - det[1:]):.2f}  applied->publish {np.median(pub[1:] - app[1:]):.2f}"
                  f"  block period {np.median(np.diff(pub)):.2f}")
