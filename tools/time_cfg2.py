import sys, time
sys.path.insert(0,'/root/repo')
import numpy as np, torch
from paper_2512_23804_b200.krylov import FgmresConfig, fgmres
from paper_2512_23804_b200.operators import steady_kkt_apply_device
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner
from paper_2512_23804_b200.problems import build_problem, steady_system
b=build_problem(2); s=steady_system(b); n=s.block_size(); shape=(s.n_h,s.n_xi)
rhs=np.zeros(3*n); rhs[:n]=np.asarray(s.mass@s.target).ravel(); bt=torch.as_tensor(rhs).cuda()
split=lambda v:[v[i*n:(i+1)*n].view(shape) for i in range(3)]
def op(v):
    o=torch.empty_like(v); steady_kkt_apply_device(s,*split(v),tuple(split(o))); return o
for ls in ('lu','fastdiag'):
    prec=build_coupled_preconditioner(s,b.partition,lead_solver=ls)
    def pr(v):
        o=torch.empty_like(v); prec.apply_device(*split(v),outs=tuple(split(o))); return o
    ts=[]
    for _ in range(4):
        torch.cuda.synchronize(); t0=time.perf_counter(); x,rep=fgmres(op,pr,bt,FgmresConfig(tol=1e-8)); torch.cuda.synchronize(); ts.append(round(time.perf_counter()-t0,4))
    # apply timing
    v=torch.randn(3*n,dtype=torch.float64,device='cuda')
    torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(5): pr(v)
    torch.cuda.synchronize(); print(ls, 'solves', ts, 'apply ms', round((time.perf_counter()-t0)/5*1e3,3), flush=True)
