"""CPU model of the Newton-3 gravity kernel's work (design tool, tools/ only): for sampled
gravity i-leaves, split into warp groups of G i-particles, replay the entry cull, the
particle cull and the survivor ring in the kernel's order, and count evaluated pairs,
useful (in-range, owned) pairs and how many (step, i-pair) evaluations could be skipped
because no lane of the step is in range of either i.  Uses the oracle's sort, leaves and
lists (test infrastructure).

  python tools/grav_sim.py [c2z] [--rows 200]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from gen import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c2z")
    ap.add_argument("--rows", type=int, default=200)
    ap.add_argument("--G", type=int, default=16)
    a = ap.parse_args()
    parts, params = make_config(a.config)
    order, keys, cellm = oracle.sort_order(parts, params)
    li = oracle.leaves(parts, params, order, cellm, 0)
    lj = oracle.leaves(parts, params, order, cellm, 1)
    L = np.asarray(params["box"])
    P = np.stack([parts[k] for k in "xyz"], 1).astype(np.float64)[order]  # sorted positions
    rc2 = params["rcut2"]
    rng = np.random.default_rng(0)
    rows = rng.choice(li["count"].shape[0], min(a.rows, li["count"].shape[0]), replace=False)
    off, col, sh = oracle.list_rows(li, lj, params, 0, rows)
    G = a.G
    st = dict(groups=0, entries=0, ent_surv=0, cand=0, surv=0, steps=0, useful=0,
              kpairs=0, skip8=0, skip1=0, half_evals=0)
    for r, ia in enumerate(rows):
        f0, c0 = li["first"][ia], li["count"][ia]
        ents = []
        for b, s in zip(col[off[r]:off[r + 1]], sh[off[r]:off[r + 1]]):
            sv = np.array([s % 3 - 1, (s // 3) % 3 - 1, s // 9 - 1]) * L
            ents.append((lj["first"][b], lj["count"][b], lj["bbox"][b, :3] + sv, lj["bbox"][b, 3:] + sv, sv))
        for g0 in range(0, c0, G):
            gs = f0 + g0
            ng = min(G, c0 - g0)
            pi = P[gs:gs + ng]
            lo, hi = pi.min(0), pi.max(0)
            st["groups"] += 1
            surv_j, surv_p = [], []
            for (jf, jc, blo, bhi, sv) in ents:
                st["entries"] += 1
                if jf + jc <= gs:
                    continue
                gap = np.maximum(0, np.maximum(blo - hi, lo - bhi))
                if (gap ** 2).sum() >= rc2 * (1 + 4e-6):
                    continue
                st["ent_surv"] += 1
                for m in range(jc):
                    j = jf + m
                    st["cand"] += 1
                    if j < gs:
                        continue
                    p = P[j] + sv
                    g = np.maximum(0, np.maximum(lo - p, p - hi))
                    if (g ** 2).sum() < rc2 * (1 + 4e-6):
                        surv_j.append(j)
                        surv_p.append(p)
            if not surv_j:
                continue
            sj = np.asarray(surv_j)
            sp = np.asarray(surv_p)
            d2 = ((sp[None, :, :] - pi[:, None, :]) ** 2).sum(-1)  # (ng, ns)
            inr = d2 < rc2
            own = ~((sj[None, :] >= gs) & (sj[None, :] < gs + ng) & (sj[None, :] <= (gs + np.arange(ng))[:, None]))
            st["useful"] += int((inr & own).sum())
            st["surv"] += sj.shape[0]
            for s0 in range(0, sj.shape[0], 32):
                blk = inr[:, s0:s0 + 32]
                st["steps"] += 1
                anyi = blk.any(1)
                anyi = np.concatenate([anyi, np.zeros(G - ng, bool)])
                for k in range(G // 2):
                    st["kpairs"] += 1
                    st["skip8"] += not (anyi[k] or anyi[k + G // 2])
                    st["skip1"] += not (anyi[2 * k] or anyi[2 * k + 1])
                # halves (i 0..G/2-1, G/2..G-1): a step evaluates a half only if some lane needs it
                st["half_evals"] += int(anyi[:G // 2].any()) + int(anyi[G // 2:].any())
            # sub-group rings: survivor copied into the ring of every sub-group (of G/Q i) whose
            # box is within r_c; each ring evaluated against its G/Q i
            for Q in (2, 4, 8):
                tot = 0
                for q in range(Q):
                    a0, a1 = q * G // Q, min((q + 1) * G // Q, ng)
                    if a0 >= ng:
                        continue
                    sub = pi[a0:a1]
                    slo, shi = sub.min(0), sub.max(0)
                    g = np.maximum(0, np.maximum(slo - sp, sp - shi))
                    nq = int(((g ** 2).sum(1) < rc2 * (1 + 4e-6)).sum())
                    tot += -(-nq // 32) * 32 * (G // Q)
                st[f"q{Q}"] = st.get(f"q{Q}", 0) + tot
    ev = st["steps"] * 32 * G
    print(f"{a.config} G={G}: groups {st['groups']}  entries/group {st['entries']/st['groups']:.0f}  "
          f"entry survivors/group {st['ent_surv']/st['groups']:.0f}  candidates/group {st['cand']/st['groups']:.0f}  "
          f"survivors/group {st['surv']/st['groups']:.0f}  steps/group {st['steps']/st['groups']:.2f}")
    print(f"  useful pairs / evaluated pair slots = {st['useful']/ev:.3f}   useful/group {st['useful']/st['groups']:.0f}")
    print(f"  skippable (step, i-pair) with pairing (k, k+G/2): {st['skip8']/st['kpairs']:.3f};  "
          f"with pairing (2k, 2k+1): {st['skip1']/st['kpairs']:.3f};  half-steps needed "
          f"{st['half_evals']/(2*st['steps']):.3f}")
    for Q in (2, 4, 8):
        print(f"  sub-group rings Q={Q}: useful / evaluated slots = {st['useful']/st[f'q{Q}']:.3f} "
              f"(evaluated {st[f'q{Q}']/ev:.3f} of Q=1)")


if __name__ == "__main__":
    main()
