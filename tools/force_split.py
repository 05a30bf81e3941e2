"""Force-split closure: short-range PP
(crk_gravity_kick, with a grid-force polynomial P5) + long-range PM (crk_pm_accel) against
the softened Newtonian force of a point mass, for P5 fitted to the analytic Gaussian-split
force (gen.configs.fit_grid_poly) and to the force the mesh actually produces
(PM.force_profile -> gen.configs.fit_poly_samples).

    python tools/force_split.py [--L 64] [--ng 64] [--json out.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from gen.configs import fit_grid_poly, fit_poly_samples, make_params, quantise  # noqa: E402
from paper_2310_16122_b200 import PM, Particles, Solver  # noqa: E402

RC, EPS2, G = 3.1, 0.01, 1.0


def probes(L, radii, n_dir, seed):
    rng = np.random.default_rng(seed)
    src = rng.random(3) * L
    u = rng.standard_normal((n_dir, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    d = (radii[None, :, None] * u[:, None, :]).reshape(-1, 3)
    pos = quantise(np.concatenate([src[None], src + d]), [L] * 3)
    return pos


def short_range(pos, L, poly):
    n = pos.shape[0]
    m = np.zeros(n, np.float32)
    m[0] = 1.0
    parts = dict(x=pos[:, 0].copy(), y=pos[:, 1].copy(), z=pos[:, 2].copy(),
                 vx=np.zeros(n, np.float32), vy=np.zeros(n, np.float32), vz=np.zeros(n, np.float32),
                 m=m, species=np.zeros(n, np.uint8), id=np.arange(n, dtype=np.int64),
                 H=np.zeros(n, np.float32), u=np.zeros(n, np.float32))
    params = make_params([L] * 3, rc=RC, eps2=EPS2, G=G, poly=poly)
    p = Particles.from_host(parts, torch.device("cuda", 0))
    s = Solver(params, 0)
    s.substep(p, 0.0, 0.0, hydro=False)
    h = p.to_host()
    s.close()
    perm = h["perm"].astype(np.int64)
    a = np.empty((n, 3))
    a[perm] = np.stack([h["ax"], h["ay"], h["az"]], 1)
    return a


def long_range(pm, pos):
    m = np.zeros(pos.shape[0])
    m[0] = 1.0
    t = [torch.tensor(v, dtype=torch.float32, device="cuda") for v in (pos[:, 0], pos[:, 1], pos[:, 2], m)]
    return torch.stack(pm.accel(*t), 1).double().cpu().numpy()


def closure(L, ng, poly_mesh, poly_ana, pm, radii, n_dir, seeds):
    rows = {"mesh": [], "analytic": []}
    rr_all = []
    for seed in seeds:
        pos = probes(L, radii, n_dir, seed)
        p64 = pos.astype(np.float64)
        d = p64[1:] - p64[0]
        d -= L * np.round(d / L)
        r = np.linalg.norm(d, axis=1)
        newton = G * r * (r * r + EPS2) ** -1.5  # toward the source
        alr = long_range(pm, pos)[1:]
        for name, poly in (("mesh", poly_mesh), ("analytic", poly_ana)):
            a = short_range(pos, L, poly)[1:] + alr
            ar = -(a * d).sum(1) / r
            at = np.linalg.norm(a - ar[:, None] * (-d / r[:, None]), axis=1)  # transverse part
            rows[name].append(np.stack([ar / newton - 1.0, at / newton], 1))
        rr_all.append(r)
    r = np.concatenate(rr_all)
    out = {}
    edges = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 2.5, 3.1, 4.0, 5.0, 6.0])
    for name in rows:
        e = np.concatenate(rows[name])
        b = []
        for lo, hi in zip(edges[:-1], edges[1:]):
            k = (r >= lo) & (r < hi)
            if k.any():
                b.append(dict(r=[float(lo), float(hi)], n=int(k.sum()),
                              rms_rel=float(np.sqrt((e[k, 0] ** 2).mean())),
                              mean_rel=float(e[k, 0].mean()),
                              max_rel=float(np.abs(e[k, 0]).max()),
                              max_transverse=float(e[k, 1].max())))
        inside = r < RC
        out[name] = dict(bins=b, rms_inside_rc=float(np.sqrt((e[inside, 0] ** 2).mean())),
                         mean_inside_rc=float(e[inside, 0].mean()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=float, default=64.0)
    ap.add_argument("--ng", type=int, default=64)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    L, ng = a.L, a.ng
    rs = RC / 4.5
    pm = PM(ng, [L] * 3, r_s=rs, G=G)
    s = np.linspace(0.0, RC * RC, 257)[1:]
    f = pm.force_profile(np.sqrt(s), n_dir=32, n_src=8, seed=1)
    poly_mesh = fit_poly_samples(s, f, RC, EPS2)
    poly_ana = fit_grid_poly(RC, EPS2)
    radii = np.linspace(0.2, 6.0, 59)
    res = closure(L, ng, poly_mesh, poly_ana, pm, radii, 24, seeds=range(4))
    res["poly_mesh"] = [float(c) for c in poly_mesh]
    res["poly_analytic"] = [float(c) for c in poly_ana]
    res["grid"] = dict(L=L, ng=ng, r_s=rs, rc=RC, eps2=EPS2)
    pm.close()
    txt = json.dumps(res, indent=1)
    print(txt)
    if a.json:
        with open(a.json, "w") as fh:
            fh.write(txt)


if __name__ == "__main__":
    main()
