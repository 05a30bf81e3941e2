"""Per-rank device time of a decomposed substep (weak scaling: c4 tiled over P ranks, as
bench.py does under torchrun), ranks emulated one after another on one GPU: for each rank,
the time of its own work (build over own + ghost particles, gravity, geometry,
corrections+extras, accel, and the pack/unpack kernels), without the transfers between
ranks.  max over ranks / the single-domain substep bounds the weak-scaling efficiency that
the exchanges' transfer time (NVLink) then lowers further.

  python tools/decomp_bench.py --P 2
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import make_config
from bench import tile_config
from paper_2310_16122_b200.domain import Decomposition, DomainRank

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
parts, params = make_config("c4")
ranks = []
for r in range(a.P):
    own, gp = tile_config(parts, params, a.P, r)
    d = Decomposition(gp, a.P)
    ranks.append(DomainRank(d, r, own, "cuda:0", outputs="forces"))
hmax2 = max(rk.local_hmax2() for rk in ranks)
h = ranks[0].d.halo_width(hmax2)
T = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {r: [] for r in range(a.P)}
for rep in range(a.reps + 1):
    sends = [rk.r1_pack(h) for rk in ranks]
    recv = [{s: sends[s][rk.r] for s in range(a.P) if rk.r in sends[s]} for rk in ranks]
    t = {}
    for rk in ranks:
        e0 = T(); e0.record()
        rk.r1_unpack_and_build(recv[rk.r])
        rk.gravity_geometry(0.0)
        e1 = T(); e1.record()
        t[rk.r] = [(e0, e1)]
    sends = [rk.r2_pack() for rk in ranks]
    for rk in ranks:
        e0 = T(); e0.record()
        rk.r2_unpack({s: sends[s][rk.r] for s in range(a.P) if rk.r in sends[s]})
        rk.corrections_extras()
        e1 = T(); e1.record()
        t[rk.r].append((e0, e1))
    sends = [rk.r3_pack() for rk in ranks]
    for rk in ranks:
        e0 = T(); e0.record()
        rk.r3_unpack({s: sends[s][rk.r] for s in range(a.P) if rk.r in sends[s]})
        rk.accel(0.0)
        e1 = T(); e1.record()
        t[rk.r].append((e0, e1))
    torch.cuda.synchronize()
    if rep > 0:
        for r in range(a.P):
            res[r].append(sum(x.elapsed_time(y) for x, y in t[r]))
print(json.dumps({"P": a.P, "ghosts_per_rank": [int(rk.n_total - rk.n_own) for rk in ranks],
                  "rank_ms": [round(sum(v) / len(v), 2) for v in res.values()]}))
