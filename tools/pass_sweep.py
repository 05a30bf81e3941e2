"""Per-pass CUDA-event times of one workload under several solver options, generated once.

  python tools/pass_sweep.py --config c4 --steps 5 "grav_kernel=0" "grav_kernel=6 nbr_cap=-1" ...
Each argument is a space-separated list of crk_params key=value settings for a fresh Solver.
"""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import make_config
from paper_2310_16122_b200 import Particles, Solver

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("variants", nargs="*", default=[""])
a = ap.parse_args()
parts, params = make_config(a.config)
passes = ["build_lists", "gravity_kick", "geometry", "corrections_extras", "hydro_accel_dudt"]
for var in a.variants:
    opts = {kv.split("=", 1)[0]: int(kv.split("=", 1)[1]) for kv in var.split()}
    p = Particles.from_host(parts, "cuda")
    s = Solver(dict(params, **opts), 0)
    st = torch.cuda.current_stream()
    ev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
          for k in passes}
    for it in range(a.steps + 2):
        for k in passes:
            if it >= 2:
                ev[k][it - 2][0].record(st)
            getattr(s, k)(p, stream=st) if k in ("build_lists", "geometry", "corrections_extras") else getattr(s, k)(p, 0.0, st)
            if it >= 2:
                ev[k][it - 2][1].record(st)
    torch.cuda.synchronize()
    ms = {k: round(sum(e0.elapsed_time(e1) for e0, e1 in ev[k]) / a.steps, 3) for k in passes}
    print(json.dumps({"variant": var, "total": round(sum(ms.values()), 2), **ms}), flush=True)
    s.close()
    del p
    torch.cuda.empty_cache()
