"""H2D throughput while the substep runs: time a 1.5 GB H2D alone and concurrently with substeps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import make_config
from paper_2310_16122_b200 import Particles, Solver

parts, params = make_config("c4")
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
p = Particles.from_host(parts, dev, outputs="forces")
q = Particles.from_host(parts, dev, outputs="forces")
torch.cuda.synchronize()
s = Solver(params, 0)
host = {k: torch.from_numpy(np.ascontiguousarray(parts[k])).pin_memory() for k in Particles.IN_F32 + ("species", "id")}
h2d = torch.cuda.Stream(dev)
for busy in (False, True, False):
    s.substep(p, stream=stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if busy:
        c0.record(stream)
        s.substep(p, stream=stream)
        s.substep(p, stream=stream)
        c1.record(stream)
    a.record(h2d)
    with torch.cuda.stream(h2d):
        q.load(host, non_blocking=True)
    b.record(h2d)
    torch.cuda.synchronize()
    print("with substeps" if busy else "alone", "H2D ms", round(a.elapsed_time(b), 2),
          "substeps ms", round(c0.elapsed_time(c1), 2) if busy else "-")
