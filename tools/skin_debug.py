import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from crk_testutil import cached_config
from paper_2310_16122_b200 import Particles, Solver
parts, params = cached_config("c1")
params["skin"] = 0.4
p = Particles.from_host(parts, "cuda")
s = Solver(params, 0)
s.substep(p)
vmag = float(np.sqrt(parts["vx"].astype(np.float64) ** 2 + parts["vy"] ** 2 + parts["vz"] ** 2).max())
dt = 0.09 / vmag
print("vmag", vmag, "dt", dt)
x0 = p.x.clone()
for k in range(4):
    s.drift(p, dt)
    torch.cuda.synchronize()
    print("drift", k, "max |dx|", float((p.x - x0).abs().max()))
    try:
        s.refresh(p); print("refresh ok")
    except Exception as e:
        print("refresh refused", e)
