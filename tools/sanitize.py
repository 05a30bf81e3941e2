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

for sym, gk, hk in ((1, 0, 0), (0, 0, 0), (1, 2, 2), (1, 1, 5)):
    parts, params = make_config("c1", symmetric=sym, grav_kernel=gk, hydro_kernel=hk)
    p = Particles.from_host(parts, "cuda")
    s = Solver(params, 0)
    s.substep(p, 0.01, 0.01)
    s.count_pairs(p)
    s.neighbour_lists(p)
    torch.cuda.synchronize()
    s.close()
# a decomposed substep (2 sub-domains emulated) in the overlapped order: ghost gravity pairs, row
# classes and crk_select_rows, the R1/R2/R3 pack/unpack kernels
from paper_2310_16122_b200.domain import Decomposition, DomainRank, substep_inprocess  # noqa: E402

parts, params = make_config("c1")
d = Decomposition(params, 2)
ranks = [DomainRank(d, r, d.split(parts, r), "cuda:0") for r in range(2)]
substep_inprocess(ranks, 0.01, 0.01, overlap=True)
torch.cuda.synchronize()
for rk in ranks:
    rk.close()
print("sanitize: substeps done")
