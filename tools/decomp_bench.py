"""Per-rank device time of a decomposed substep (weak scaling: c4 tiled over P ranks, as
bench.py does under torchrun), ranks emulated one after another on one GPU with the exchange
protocol of domain.substep_dist (persistent plan, device counts, one count readback): for each
rank, the time of its own work — R1 selection and packing, unpack + build over own + ghost
particles, gravity, geometry, R2 pack/unpack, corrections+extras, R3 pack/unpack, accel —
without the transfers between ranks.  max over ranks / the single-domain substep bounds the
weak-scaling efficiency that the transfers' time (NVLink) then lowers further.

  python tools/decomp_bench.py --P 8 [--config c4] [--reps 3]
(P = 8 at c4 per rank fits one GPU's memory only with --no-carry; or --config lat:128,128,128:0.1:16522)
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from gen import make_config  # noqa: E402
from bench import tile_config  # noqa: E402
from paper_2310_16122_b200.domain import Decomposition, DomainRank, EmuExchange  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--config", default="c4")
ap.add_argument("--min-free-gb", type=float, default=12.0)
ap.add_argument("--no-carry", action="store_true",
                help="do not carry the own sets (no spare local-set buffer: eight c4-sized ranks then fit one "
                     "GPU; the build sorts the random-order own set every substep, an upper bound)")
a = ap.parse_args()
parts, params = make_config(a.config)
ranks = []
for r in range(a.P):
    own, gp = tile_config(parts, params, a.P, r)
    d = Decomposition(gp, a.P)
    ranks.append(DomainRank(d, r, own, "cuda:0", outputs="forces"))
hmax2 = max(rk.local_hmax2() for rk in ranks)
h = ranks[0].d.halo_width(hmax2)
for rk in ranks:
    rk.plan(h)
T = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {r: [] for r in range(a.P)}
phases = {r: [] for r in range(a.P)}
ex = EmuExchange(ranks)


def phase(t, rk, fn):
    e0 = T()
    e0.record()
    out = fn()
    e1 = T()
    e1.record()
    t[rk.r].append((e0, e1))
    return out


for rep in range(a.reps + 1):
    t = {r: [] for r in range(a.P)}
    cs = [phase(t, rk, rk.r1_select_pack) for rk in ranks]
    for rk in ranks:
        for q, s in enumerate(rk.peers):
            rk.cnt_recv[q].copy_(cs[s][ranks[s].peers.index(rk.r)])
    for rk in ranks:
        rk.r1_sizes(np.stack([rk.cnt_send.cpu().numpy(), rk.cnt_recv.cpu().numpy()]))
    msgs = [rk.r1_messages() for rk in ranks]
    ex.exchange_all([m[0] for m in msgs], [m[1] for m in msgs])
    for rk in ranks:
        phase(t, rk, rk.r1_unpack)
        phase(t, rk, lambda: rk.solver.build_lists(rk.p, rk.stream))
        phase(t, rk, rk._gas_idx)
        phase(t, rk, lambda: rk.solver.gravity_kick(rk.p, 0.0, rk.stream))
        phase(t, rk, lambda: rk.solver.geometry(rk.p, rk.stream))
        free = torch.cuda.mem_get_info()[0] / 2**30
        if free < a.min_free_gb:
            raise SystemExit(f"device memory nearly exhausted after rank {rk.r} ({free:.1f} GB free): use a smaller config")
    msgs = [phase(t, rk, rk.r2_messages) for rk in ranks]
    ex.exchange_all([m[0] for m in msgs], [m[1] for m in msgs])
    for rk, m in zip(ranks, msgs):
        phase(t, rk, lambda: (rk.r2_unpack(m[1]), rk.corrections_extras()))
    msgs = [phase(t, rk, rk.r3_messages) for rk in ranks]
    ex.exchange_all([m[0] for m in msgs], [m[1] for m in msgs])
    for rk, m in zip(ranks, msgs):
        phase(t, rk, lambda: (rk.r3_unpack(m[1]), rk.accel(0.0)))
    if not a.no_carry:
        for rk in ranks:
            phase(t, rk, rk.carry_own)
    torch.cuda.synchronize()
    if rep > 0:
        for r in range(a.P):
            res[r].append(sum(x.elapsed_time(y) for x, y in t[r]))
            phases[r].append([x.elapsed_time(y) for x, y in t[r]])
msg_bytes = [int(sum(rk.n_send.values()) * 48 + sum(rk.g_send.values()) * (16 + 144)) for rk in ranks]
print(json.dumps({"P": a.P, "config": a.config, "carry_own": not a.no_carry, "halo_cells": h,
                  "ghosts_per_rank": [int(rk.n_total - rk.n_own) for rk in ranks],
                  "bytes_sent_per_rank": msg_bytes,
                  "rank_ms": [round(sum(v) / len(v), 2) for v in res.values()],
                  "max_rank_ms": round(max(sum(v) / len(v) for v in res.values()), 2),
                  "phase_names": ["r1 select+pack", "r1 unpack", "build", "gas idx", "gravity", "geometry", "r2 pack",
                                  "r2 unpack+cor/ext", "r3 pack", "r3 unpack+accel", "carry own"],
                  "rank_phase_ms": [[round(float(x), 2) for x in np.median(np.asarray(v), 0)] for v in phases.values()]}))
