import sys
sys.path.insert(0,'/root/repo')
import numpy as np, torch
from paper_2512_23804_b200.preconditioners import build_coupled_preconditioner, build_steady_preconditioner
from paper_2512_23804_b200.operators import steady_kkt_apply_device
from paper_2512_23804_b200.problems import build_problem, steady_system
b=build_problem(5); s=steady_system(b); shape=(s.n_h,s.n_xi)
blocks=[torch.randn(shape,dtype=torch.float64,device='cuda') for _ in range(3)]
outs=tuple(torch.empty_like(blocks[0]) for _ in range(3))
def timed(fn,reps=10):
    fn(); torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize(); return e0.elapsed_time(e1)/reps
for name,prec in (('hgsoc',build_coupled_preconditioner(s,b.partition,lead_solver='fastdiag')),('blockdiag',build_steady_preconditioner(s,b.partition,'cheb5',lead_solver='fastdiag'))):
    f=lambda: prec.apply_device(*blocks, outs=outs)
    t_eager=timed(f)
    # warm on a side stream then capture
    st=torch.cuda.Stream(); st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for _ in range(2): f()
    torch.cuda.current_stream().wait_stream(st); torch.cuda.synchronize()
    g=torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    ref=[o.clone() for o in outs]
    t_graph=timed(g.replay)
    f(); torch.cuda.synchronize()
    err=max(float((o-r).abs().max()) for o,r in zip(outs,ref))
    print(name,'eager %.3f ms graph %.3f ms  maxdiff %.1e'%(t_eager,t_graph,err), flush=True)
t=timed(lambda: steady_kkt_apply_device(s,*blocks,outs)); print('kkt eager %.3f'%t)
