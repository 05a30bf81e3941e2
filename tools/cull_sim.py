"""CPU model of the pair kernels' culling: for each i-leaf and warp group of G i-particles,
count staged candidates, bbox survivors, warp steps and useful pairs (gravity / hydro).
Uses the oracle's leaves and lists (test infrastructure; tools/ only)."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from gen import make_config

def sim(name, G_grav=(16, 8), G_hyd=(8, 4), max_leaves=300, **kw):
    parts, params = make_config(name, **kw)
    order, keys, cellm = oracle.sort_order(parts, params)
    ls = [oracle.leaves(parts, params, order, cellm, k) for k in range(4)]
    L = np.asarray(params["box"])
    P = np.stack([parts[k] for k in "xyz"], 1).astype(np.float64)
    gas_sorted = order[parts["species"][order] == 1]
    H2 = (parts["H"] * parts["H"]).astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(0)
    for mode, (ki, kj, mem, Gs) in enumerate([(0, 1, order, G_grav), (2, 3, gas_sorted, G_hyd)]):
        la, lb = ls[ki], ls[kj]
        rows = rng.choice(la["count"].shape[0], min(max_leaves, la["count"].shape[0]), replace=False)
        off, col, sh = oracle.list_rows(la, lb, params, mode, rows)
        for G in Gs:
            S = 32 // G
            tot = dict(cand=0, surv=0, steps=0, useful=0, iparts=0, warps=0)
            for r, a in enumerate(rows):
                ii = mem[la["first"][a]: la["first"][a] + la["count"][a]]
                cand = []
                for b, s in zip(col[off[r]:off[r+1]], sh[off[r]:off[r+1]]):
                    jj = mem[lb["first"][b]: lb["first"][b] + lb["count"][b]]
                    sv = np.array([s % 3 - 1, (s // 3) % 3 - 1, s // 9 - 1]) * L
                    cand.append((jj, P[jj] + sv))
                cj = np.concatenate([c[0] for c in cand]); cp = np.concatenate([c[1] for c in cand])
                tot["cand"] += cj.shape[0]
                for g0 in range(0, ii.shape[0], G):
                    gi = ii[g0:g0+G]; pi = P[gi]
                    lo, hi = pi.min(0), pi.max(0)
                    gap = np.maximum(0, np.maximum(lo - cp, cp - hi))
                    d2 = (gap**2).sum(1)
                    if mode == 0:
                        keep = d2 < params["rcut2"] * (1 + 4e-6)
                    else:
                        keep = d2 < np.maximum(H2[gi].max(), H2[cj]) * (1 + 4e-6)
                    sj = cj[keep]; sp = cp[keep]
                    tot["surv"] += sj.shape[0]; tot["steps"] += -(-sj.shape[0] // S); tot["warps"] += 1
                    tot["iparts"] += gi.shape[0]
                    d = sp[None, :, :] - pi[:, None, :]
                    s2 = (d**2).sum(-1)
                    if mode == 0:
                        u = (s2 < params["rcut2"]) & (sj[None, :] != gi[:, None])
                    else:
                        u = (s2 < np.maximum(H2[gi][:, None], H2[sj][None, :])) & (sj[None, :] != gi[:, None])
                    tot["useful"] += int(u.sum())
            lanes = tot["steps"] * 32
            print(f"{name} {'grav' if mode==0 else 'hydro-sym'} G={G}: cand/CTA {tot['cand']/len(rows):.0f} "
                  f"surv/warp {tot['surv']/tot['warps']:.0f} useful/i {tot['useful']/tot['iparts']:.1f} "
                  f"useful/lane-slot {tot['useful']/lanes:.3f} lane-slots per i {lanes/tot['iparts']:.0f}")

if __name__ == "__main__":
    sim(sys.argv[1] if len(sys.argv) > 1 else "c2z")
