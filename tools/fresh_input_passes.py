"""Per-pass times of a substep on freshly loaded (generator random order) inputs vs on the
previous step's in-place sorted order."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import make_config
from paper_2310_16122_b200 import Particles, Solver

parts, params = make_config("c4")
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
p = Particles.from_host(parts, dev, outputs="forces")
torch.cuda.synchronize()
s = Solver(params, 0)
host = {k: torch.from_numpy(np.ascontiguousarray(parts[k])).pin_memory() for k in Particles.IN_F32 + ("species", "id")}
passes = ["build_lists", "gravity_kick", "geometry", "corrections_extras", "hydro_accel_dudt"]
for fresh in (False, True, False, True):
    if fresh:
        p.load(host)
        torch.cuda.synchronize()
    ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in passes}
    for k in passes:
        ev[k][0].record(st)
        f = getattr(s, k)
        f(p, stream=st) if k in ("build_lists", "geometry", "corrections_extras") else f(p, 0.0, st)
        ev[k][1].record(st)
    torch.cuda.synchronize()
    print("fresh" if fresh else "sorted", {k: round(ev[k][0].elapsed_time(ev[k][1]), 2) for k in passes})
