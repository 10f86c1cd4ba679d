cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 800 python tools/ab_variants.py shipped:SGKKT_S9_TMA=1 c4:SGKKT_S9_TMA=1 > gpurun_out/g43_ab.log 2>&1
cat gpurun_out/g43_ab.log
timeout 600 python tools/time_kkt.py 5 > gpurun_out/g43_kkt.log 2>&1; tail -5 gpurun_out/g43_kkt.log
timeout 600 python - > gpurun_out/g43_kktstats.log 2>&1 <<'PY'
from paper_2512_23804_b200.problems import build_problem, steady_system
b = build_problem(5); s = steady_system(b)
p = s.kkt_program()
f = p.fast9(s.pattern.n_slices)
print(f.host.stats if f is not None else None)
PY
tail -3 gpurun_out/g43_kktstats.log
timeout 600 python tools/time_matvec.py 3 > gpurun_out/g43_cfg3.log 2>&1; tail -3 gpurun_out/g43_cfg3.log
