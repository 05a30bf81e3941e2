"""Variant portfolio: per-pass times of every kernel variant on one
workload, each pass's efficiency e = t_best / t_variant (the form of the paper's per-kernel
efficiency figures, §5.4 Figs. optimized-*), and, per portfolio (one variant choice
for every pass), the harmonic mean of the efficiencies over the passes — Eq. 1 (PAPER.md:
172-182) taken across kernels instead of platforms, since there is one platform here.

  python tools/variant_portfolio.py [--config c4] [--out profiles/r01/variant_portfolio.json]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import make_config
from paper_2310_16122_b200 import Particles, Solver

PORTFOLIOS = {
    "lists + pipelined Newton-3 gravity (default)": {},
    "lists, CTA-staged Newton-3 gravity": {"grav_kernel": 7},
    "lists, warp gravity without pipeline": {"grav_kernel": 6},
    "lists, half-warp shuffle gravity (the paper's algorithm)": {"grav_kernel": 8},
    "lists, Newton-3 accel": {"hydro_kernel": 5},
    "lists, corrections + extras in one walk (moment form)": {"hydro_kernel": 2},
    "lists, gravity with 4 CTAs/SM and 32 staged leaves": {"grav_kernel": 1},
    "lists, accel with 8 lanes per i (one 16-warp CTA per SM)": {"hydro_kernel": 4},
    "lists, accel with 8 lanes per i, 128-entry staging rounds": {"hydro_kernel": 6},
    "on-the-fly culling everywhere (no neighbour lists)": {"nbr_cap": -1, "grav_kernel": 7},
}
PASSES = ["build_lists", "gravity_kick", "geometry", "corrections_extras", "hydro_accel_dudt"]

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--out", default="gpurun_out/variant_portfolio.json")
a = ap.parse_args()
parts, params = make_config(a.config)
times = {}
for name, opts in PORTFOLIOS.items():
    p = Particles.from_host(parts, "cuda", outputs="forces")
    s = Solver(dict(params, **opts), 0)
    st = torch.cuda.current_stream()
    ev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
          for k in PASSES}
    for it in range(a.steps + 2):
        for k in PASSES:
            if it >= 2:
                ev[k][it - 2][0].record(st)
            f = getattr(s, k)
            f(p, stream=st) if k in ("build_lists", "geometry", "corrections_extras") else f(p, 0.0, st)
            if it >= 2:
                ev[k][it - 2][1].record(st)
    torch.cuda.synchronize()
    times[name] = {k: sum(e0.elapsed_time(e1) for e0, e1 in ev[k]) / a.steps for k in PASSES}
    s.close()
    del p
    torch.cuda.empty_cache()
best = {k: min(t[k] for t in times.values()) for k in PASSES}
res = {}
for name, t in times.items():
    eff = {k: best[k] / t[k] for k in PASSES}
    res[name] = {"ms": {k: round(v, 3) for k, v in t.items()}, "total_ms": round(sum(t.values()), 3),
                 "efficiency": {k: round(v, 3) for k, v in eff.items()},
                 "harmonic_mean_efficiency": round(len(PASSES) / sum(1.0 / v for v in eff.values()), 3)}
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
json.dump({"config": a.config, "portfolios": res}, open(a.out, "w"), indent=1)
for name, r in res.items():
    print(f"{r['harmonic_mean_efficiency']:.3f}  {r['total_ms']:8.2f} ms  {name}  {r['efficiency']}")
