"""One short-range substep of config 1 (+ the count mode) for compute-sanitizer (SURVEY.md §5:
memcheck / racecheck / synccheck on config 1 — the cp.async and mbarrier staging of the pair
kernels, the warp-synchronous rings, the Newton-3 atomics).

  compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from gen import make_config  # noqa: E402
from paper_2310_16122_b200 import Particles, Solver  # noqa: E402

for sym, gk, hk in ((1, 0, 0), (0, 0, 0), (1, 2, 2)):
    parts, params = make_config("c1", symmetric=sym, grav_kernel=gk, hydro_kernel=hk)
    p = Particles.from_host(parts, "cuda")
    s = Solver(params, 0)
    s.substep(p, 0.01, 0.01)
    s.count_pairs(p)
    s.neighbour_lists(p)
    torch.cuda.synchronize()
    s.close()
print("sanitize: substeps done")
