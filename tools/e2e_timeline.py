"""Timeline of the pipelined e2e loop: per step, H2D start/end and compute start/end (ms from t0)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import make_config
from paper_2310_16122_b200 import Particles, Solver

parts, params = make_config("c4")
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
sets = [Particles.from_host(parts, dev, outputs="forces"), Particles.from_host(parts, dev, outputs="forces")]
torch.cuda.synchronize()
solver = Solver(params, 0)
host = {k: torch.from_numpy(np.ascontiguousarray(parts[k])).pin_memory() for k in Particles.IN_F32 + ("species", "id")}
h2d = torch.cuda.Stream(dev)
T = lambda: torch.cuda.Event(enable_timing=True)
N = 6
t0 = T(); t0.record(stream)
hs, he, cs, ce, hostt = [], [], [], [], []
ev_in = [torch.cuda.Event(), torch.cuda.Event()]
ev_done = [torch.cuda.Event(), torch.cuda.Event()]
h2d.wait_stream(stream)
a, b_ = T(), T(); a.record(h2d)
with torch.cuda.stream(h2d):
    sets[0].load(host, non_blocking=True)
b_.record(h2d); ev_in[0].record(h2d); hs.append(a); he.append(b_)
w0 = time.perf_counter()
for k in range(N):
    b = k % 2
    stream.wait_event(ev_in[b])
    c0, c1 = T(), T()
    c0.record(stream)
    solver.substep(sets[b], stream=stream)
    c1.record(stream)
    hostt.append(round((time.perf_counter() - w0) * 1e3, 1))
    cs.append(c0); ce.append(c1)
    ev_done[b].record(stream)
    if k + 1 < N:
        nb = (k + 1) % 2
        if k >= 1:
            h2d.wait_event(ev_done[nb])
        a, b_ = T(), T(); a.record(h2d)
        with torch.cuda.stream(h2d):
            sets[nb].load(host, non_blocking=True)
        b_.record(h2d); ev_in[nb].record(h2d); hs.append(a); he.append(b_)
torch.cuda.synchronize()
f = lambda e: round(t0.elapsed_time(e), 1)
for k in range(N):
    print(f"step {k}: H2D [{f(hs[k])}, {f(he[k])}]  compute [{f(cs[k])}, {f(ce[k])}]  host returned from substep at {hostt[k]} ms")
