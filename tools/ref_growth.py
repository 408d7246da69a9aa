"""The UNMODIFIED reference (oracle/_ref) on the C2 physics (extremal Kerr
a=M, s=-2, m=2, its own ell=2 initial data), 2048x16, reference mixed: max|u|
after 1000 / 3000 / 6000 SSP-RK3 steps.  The pulse grows exponentially in
the reference as on the GPU tiers (tools/probe_growth.py); bench.py's
sustained phase restarts it on small grids."""
import sys, numpy as np, time
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle as O
phys=O.Physics(a=1.0, spin=-2, mmode=2, ell=2, center=1.0, width=0.22)
ref=O.RefSolver(phys, 2048, 16, mode="mixed", workers=8)
u,lo=ref.initial_data()
dt=ref.select_dt("ssprk33")
s=0
for k in (1000,2000,3000,4000):
    t=time.time()
    (u,lo),st,per=ref.advance_timed(u,lo,dt,s,s+k); s+=k
    print(s, s*dt[0] if hasattr(dt,'__len__') else s*dt, np.abs(u).max(), st, time.time()-t, flush=True)
