"""Diagnose the e2e pipeline: substeps with and without the per-step H2D / D2H copies overlapped."""
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
outk = ["ax", "ay", "az", "ahx", "ahy", "ahz", "dudt", "perm"]
hout2 = [{k: torch.empty(sets[0].n, dtype=getattr(sets[0], k).dtype).pin_memory() for k in outk} for _ in range(2)]
h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
ev_in = [torch.cuda.Event(), torch.cuda.Event()]
ev_done = [torch.cuda.Event(), torch.cuda.Event()]
ev_out = [torch.cuda.Event(), torch.cuda.Event()]

def run(nsteps, do_in, do_out):
    h2d.wait_stream(stream)
    if do_in:
        with torch.cuda.stream(h2d):
            sets[0].load(host, non_blocking=True)
    ev_in[0].record(h2d)
    for k in range(nsteps):
        b = k % 2
        stream.wait_event(ev_in[b])
        if k >= 2:
            stream.wait_event(ev_out[b])
        solver.substep(sets[b], stream=stream)
        ev_done[b].record(stream)
        if k + 1 < nsteps:
            nb = (k + 1) % 2
            if k >= 1:
                h2d.wait_event(ev_done[nb])
            if do_in:
                with torch.cuda.stream(h2d):
                    sets[nb].load(host, non_blocking=True)
            ev_in[nb].record(h2d)
        d2h.wait_event(ev_done[b])
        if do_out:
            with torch.cuda.stream(d2h):
                for key in outk:
                    hout2[b][key].copy_(getattr(sets[b], key), non_blocking=True)
        ev_out[b].record(d2h)
    stream.wait_stream(d2h)

for do_in, do_out in [(False, False), (True, False), (False, True), (True, True)]:
    run(2, do_in, do_out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record(stream)
    run(6, do_in, do_out)
    e1.record(stream)
    torch.cuda.synchronize()
    print("in", do_in, "out", do_out, "ms/step", round(e0.elapsed_time(e1) / 6, 2), "wall", round((time.perf_counter() - t) / 6 * 1e3, 2))
