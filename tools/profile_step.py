"""One short-range substep under cudaProfilerStart/Stop, for ncu (--profile-from-start off).

  ncu --profile-from-start off ... python tools/profile_step.py --config c4 [--warmup 2]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import make_config
from paper_2310_16122_b200 import Particles, Solver

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--set", nargs="*", default=[], help="crk_params overrides k=v")
a = ap.parse_args()
parts, params = make_config(a.config)
p = Particles.from_host(parts, "cuda", outputs="forces")  # as bench.py
s = Solver(dict(params, **{kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.set}), 0)
for _ in range(a.warmup):
    s.substep(p)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.steps):
    s.substep(p)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("profiled", a.steps, "substep(s) of", a.config, "launches/ctx", s.launch_count())
