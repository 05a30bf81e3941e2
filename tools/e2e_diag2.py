"""Do concurrent D2H copies slow the substep's kernels (L2 pollution)?  Per-pass times with a
background D2H stream copying 1 GB in a loop vs without."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import make_config
from paper_2310_16122_b200 import Particles, Solver

parts, params = make_config("c4")
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
p = Particles.from_host(parts, dev, outputs="forces")
torch.cuda.synchronize()
s = Solver(params, 0)
n = p.n
hout = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(8)]
dsrc = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(8)]
ds = torch.cuda.Stream(dev)
passes = ["build_lists", "gravity_kick", "geometry", "corrections_extras", "hydro_accel_dudt"]
for bg in (False, True, False):
    for _ in range(2):
        s.substep(p, stream=stream)
    torch.cuda.synchronize()
    if bg:
        with torch.cuda.stream(ds):
            for _ in range(12):
                for x, y in zip(hout, dsrc): x.copy_(y, non_blocking=True)
    ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in passes}
    for k in passes:
        ev[k][0].record(stream)
        f = getattr(s, k)
        f(p, stream=stream) if k in ("build_lists", "geometry", "corrections_extras") else f(p, 0.0, stream)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    print("background D2H" if bg else "alone", {k: round(ev[k][0].elapsed_time(ev[k][1]), 2) for k in passes})
