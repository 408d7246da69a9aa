"""Growth of the extremal-Kerr m=2 pulse on the device-assembled planes
(paper_2010_04760_b200/planes.py): max |u| after 100 .. 161100 SSP-RK3 steps
on 2048x64 and 4096x128, fast tiers.  Shows why bench.py's sustained phase
restarts the pulse every tau = 20 on small grids.

    python tools/probe_growth.py > gpurun_out/probe_growth.txt
"""
import sys, numpy as np, torch
sys.path.insert(0,'.')
from paper_2010_04760_b200 import hwgpu, planes, synthetic
for (n,nt) in ((2048,64),(4096,128)):
  for mode in ("mixed","f64"):
    prob = planes.problem(n, nt)
    g = hwgpu.GpuEvolution(n, nt, prob["drho"], prob["dtheta"], prob["parity"], prob["coef"], prob["cotth"], hwgpu.SchemeSpec("weno5", mode))
    g.set_state(synthetic.initial_state(prob))
    dt = synthetic.select_dt(prob)
    s=0; res=[]
    for chunk in (100,1000,10000,50000,100000):
        g.launch_steps("ssprk33", dt, s, chunk); s+=chunk
        torch.cuda.synchronize()
        b, bs = g.status()
        u = g.get_state()
        res.append((s, b, bs, float(np.abs(u).max())))
        if b: break
    print(n, nt, mode, "dt", dt, "maxspeed", prob["max_speed"], res, flush=True)
    g.close()
