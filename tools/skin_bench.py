"""Sub-cycle force evaluation with and without list reuse on c4: a full substep (build +
passes) with skin 0 and with a skin, and refresh + passes on the skin lists after a drift."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import make_config
from paper_2310_16122_b200 import Particles, Solver

parts, params0 = make_config("c4")
st = torch.cuda.current_stream()
T = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
out = {}
for skin in (0.0, 0.3):
    params = dict(params0, skin=skin)
    p = Particles.from_host(parts, "cuda", outputs="forces")
    s = Solver(params, 0)
    for _ in range(2):
        s.substep(p)
    e0, e1 = T(), T()
    e0.record(st)
    for _ in range(3):
        s.substep(p)
    e1.record(st)
    torch.cuda.synchronize()
    out[f"substep (build + passes), skin {skin}"] = e0.elapsed_time(e1) / 3
    if skin > 0:
        vmag = float(torch.sqrt(p.vx ** 2 + p.vy ** 2 + p.vz ** 2).max())
        dt = 0.02 / vmag
        ms = []
        for _ in range(3):
            s.drift(p, dt)
            e0, e1 = T(), T()
            e0.record(st)
            s.refresh(p)
            s.substep(p, build=False)
            e1.record(st)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        out[f"refresh + passes, skin {skin}"] = sum(ms) / len(ms)
    s.close()
    del p
    torch.cuda.empty_cache()
print(json.dumps({k: round(v, 2) for k, v in out.items()}))
