"""Regenerate DESIGN.md §5's final-line paragraph and time-to-solution table
from profiles/bench_r02_final.json (+ the reference arm line): every number in
the section then traces to the committed bench line.
python tools/design_numbers.py [--write]  (rewrites the block between the
<!-- bench:begin --> / <!-- bench:end --> markers in DESIGN.md)"""
import json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
d = json.loads((ROOT / "profiles" / "bench_r02_final.json").read_text())
ref = json.loads((ROOT / "profiles" / "bench_r02_reference_arm.json").read_text())
s, rf, cb = d["solves"], d["roofline"], d["cpu_baseline"]
ab = s["cfg5_apply_breakdown"]
cpu5 = cb["solves"]["cfg5"]["beta=0.01"]
refc = cpu5["reference_sgkkt_build_container"]
ref_solve = ref.get("solves", {}).get("cfg5", {})
def fmt(v, key):
    e = v.get(key)
    return f"{e['iterations']} / {e['seconds']:.3f}" if e else "—"
lines = []
lines.append(
    f"Final line (`profiles/bench_r02_final.json`, one B200 at {d['clocks']['sm_mhz']:.0f} MHz, throttle reasons "
    f"{d['clocks']['reasons'] or 'none'}): **value {d['value']:.1f} GB/s** = {d['ms_per_step']:.3f} ms per config-4 "
    f"matvec, roofline frac **{rf['frac']:.4f}** of the measured {rf['peak']:.1f} GB/s (DRAM traffic per launch "
    f"{rf['traffic'] / 1e9:.3f} GB = {rf['traffic'] / 1095340704:.2f}·B), fp64 {rf['fp64_tflops']:.2f} TF "
    f"({rf['fp64_frac']:.3f} of DFMA); **e2e {d['e2e']['value']:.1f} GB/s** through `kron_apply` on pinned host "
    f"buffers ({d['e2e']['pcie_roofline']['frac_of_duplex_copy_time']:.2f} of the box's duplex PCIe copy time); CPU "
    f"port {cb['value']:.3f} GB/s ({cb['cores']} core; reference arm `profiles/bench_r02_reference_arm.json` "
    f"{ref['value']:.3f} GB/s).  Config-5 KKT matvec {ab['kkt_matvec_ms']:.3f} ms ({ab['kkt_hbm_frac']:.3f} of HBM); "
    f"hGSoc apply LU {ab['hgsoc_lu']['apply_ms']:.1f} ms, fastdiag {ab['hgsoc_fastdiag']['apply_ms']:.2f} ms; CPU "
    f"sample on the box host: one oracle-port hGSoc apply {cpu5['hgsoc_apply_s']:.1f} s + KKT matvec "
    f"{cpu5['kkt_matvec_s']:.1f} s per FGMRES iteration.")
lines.append("")
lines.append("Time to solution (tol 1e-8 unless stated; warm; setup — host SuperLU factorisation, device tables — "
             "reported separately in the line):")
lines.append("")
lines.append("| config | solver | GPU LU: its / s | GPU fastdiag: its / s | CPU (1 core): its / s |")
lines.append("|---|---|---|---|---|")
c1, c3, c2 = s["cfg1_forward"], s["cfg3_forward"], s["cfg2"]["beta=0.01"]
lines.append(f"| 1 (forward) | hGS-CG, n_τ = 5 | {fmt(c1, 'hgs_cg n_tau=5')} | {fmt(c1, 'hgs_cg[fastdiag] n_tau=5')} | — |")
CPU3 = {1: "sgkkt sweep + matvec, oracle CG: 26 / 186.2", 7: "10 / 71.0", 924: "8 / 80.0"}
for nt in (1, 7, 924):
    lines.append(f"| 3 (forward, 924 terms) | hGS-CG, n_τ = {nt} | {fmt(c3, f'hgs_cg n_tau={nt}')} | "
                 f"{fmt(c3, f'hgs_cg[fastdiag] n_tau={nt}')} | {CPU3[nt]} |")
ref2 = ref.get("solves", {}).get("cfg2", {}).get("beta=0.01", {})
def refs(k):
    e = ref2.get(k)
    return f"{e['iterations']} / {e['seconds']:.1f} (port)" if e else "—"
lines.append(f"| 2, β=1e-2 | hGSoc-FGMRES | {fmt(c2, 'hgsoc_fgmres')} | {fmt(c2, 'hgsoc_fgmres[fastdiag]')} | {refs('hgsoc_fgmres')} |")
lines.append(f"| 2, β=1e-2 | block-diag hGS MINRES | {fmt(c2, 'blockdiag_hgs_minres')} | "
             f"{fmt(c2, 'blockdiag_hgs_minres[fastdiag]')} | {refs('blockdiag_hgs_minres')} |")
for beta, lab in (("beta=0.01", "1e-2"), ("beta=0.0001", "1e-4"), ("beta=1e-06", "1e-6")):
    v = s["cfg5"][beta]
    r = refc[beta]
    extra = ""
    e = ref_solve.get(beta, {}).get("hgsoc_fgmres") if isinstance(ref_solve, dict) else None
    if e:
        extra = f"; port on the GPU box host {e['iterations']} / {e['seconds']:.1f}"
    lines.append(f"| 5, β={lab} | hGSoc-FGMRES | {fmt(v, 'hgsoc_fgmres')} | {fmt(v, 'hgsoc_fgmres[fastdiag]')} | "
                 f"sgkkt: {r['hgsoc_fgmres']['iterations']} / {r['hgsoc_fgmres']['seconds']}{extra} |")
    lines.append(f"| 5, β={lab} | block-diag hGS MINRES | {fmt(v, 'blockdiag_hgs_minres')} | "
                 f"{fmt(v, 'blockdiag_hgs_minres[fastdiag]')} | sgkkt ops + oracle MINRES: "
                 f"{r['blockdiag_hgs_minres']['iterations']} / {r['blockdiag_hgs_minres']['seconds']} |")
td = s["time_dependent"]
lines.append(f"| time-dep. (3,3) N_t={td['n_t']}, {td['dofs'] // 1000}k DoF, tol 1e-6 | PINT-FGMRES | "
             f"{td['gpu']['iterations']} / {td['gpu']['seconds']:.3f} | {td['gpu[fastdiag]']['iterations']} / "
             f"{td['gpu[fastdiag]']['seconds']:.3f} | — |")
block = "\n".join(lines)
if "--write" in sys.argv:
    p = ROOT / "DESIGN.md"
    t = p.read_text()
    a, b = t.index("<!-- bench:begin -->"), t.index("<!-- bench:end -->")
    p.write_text(t[:a] + "<!-- bench:begin -->\n" + block + "\n" + t[b:])
else:
    print(block)
