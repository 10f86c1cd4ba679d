"""cProfile of the host side of one time-dependent preconditioner apply (fastdiag leads)."""
import cProfile, pstats, runpy, sys
sys.argv = ["tools/time_timedep.py"]
src = open("tools/time_timedep.py").read().split("for ls in")[0]
g = {"__name__": "x", "__file__": "tools/time_timedep.py"}
exec(compile(src, "tools/time_timedep.py", "exec"), g)
prec = g["build_time_preconditioner"](g["sys_"], g["b"].partition, "cheb5", lead_solver="fastdiag")
bd, out = g["bd"], g["out"]
prec.apply_device(bd, out)
import torch; torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(5): prec.apply_device(bd, out)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
