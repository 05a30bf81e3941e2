"""One build_lists on freshly loaded (random order) inputs under cudaProfilerStart/Stop (ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import make_config
from paper_2310_16122_b200 import Particles, Solver

parts, params = make_config("c4")
p = Particles.from_host(parts, "cuda", outputs="forces")
s = Solver(params, 0)
s.substep(p)
p.load(parts)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
s.build_lists(p)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
