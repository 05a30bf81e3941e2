"""Count mode of the PRODUCTION kernels and the exact gas neighbour lists (GPU, C-ABI).

SURVEY.md §4 / SPEC.md:374-382 (integer-payload audit: every pair once per direction) and
PAPER.md:418 (§5.3: pair-wise symmetry is "critically important for the correctness").
crk_count_pairs runs integer-payload instantiations of the kernels the force passes run —
the Newton-3 pipelined gravity kernel (both directions from one evaluation, reactions by
atomics, the own-group and ghost rules) and the neighbour-list walks of corrections/extras
and accel/du-dt — so exact counts prove that those kernels visit exactly the O2 pairs, which
a force sum cannot show near r_c (where the continuity-constrained pair force vanishes).
"""
import numpy as np
import pytest

import oracle
from crk_testutil import cached_config, run_gpu

pytestmark = pytest.mark.gpu


def _gpu_lists(parts, params, cap_out=160):
    import torch
    from paper_2310_16122_b200 import Particles, Solver

    p = Particles.from_host(parts, torch.device("cuda", 0))
    s = Solver(params, 0)
    s.build_lists(p)
    s.geometry(p)
    cnt, nbr = s.neighbour_lists(p, cap_out)
    cg, ch, cs = s.count_pairs(p)
    torch.cuda.synchronize()
    perm = p.perm.cpu().numpy().astype(np.int64)
    out = dict(cnt=cnt.cpu().numpy(), nbr=nbr.cpu().numpy(), perm=perm,
               counts=tuple(c.cpu().numpy() for c in (cg, ch, cs)))
    s.close()
    return out


@pytest.mark.parametrize("name", ["c1", "lat:32,16,16:0.1:3", "c2z"])
def test_neighbour_lists_equal_oracle_sets(name):
    """Every gas particle's list (built by the geometry kernel) holds exactly itself and the
    gas particles j with s32 < max(H_i^2, H_j^2) (oracle.neighbour_sets, pred 2), and the
    list-walk counts equal the oracle's gather / symmetric counts."""
    parts, params = cached_config(name)
    g = _gpu_lists(parts, params)
    perm = g["perm"]
    n = perm.shape[0]
    gas_sorted = np.nonzero(parts["species"][perm] == 1)[0]
    assert np.all(g["cnt"][gas_sorted] >= 1), "complete lists (capacity 128 on these inputs)"
    tg = perm[gas_sorted]  # input indices of the gas particles, in sorted order
    off, ref = oracle.neighbour_sets(parts, params, tg, 2)
    sym_len = np.diff(off)
    assert np.array_equal(g["cnt"][gas_sorted], sym_len + 1)
    for r, i_sorted in enumerate(gas_sorted):
        got = np.sort(perm[g["nbr"][i_sorted, : g["cnt"][i_sorted]]])
        exp = np.sort(np.concatenate([ref[off[r]:off[r + 1]], [perm[i_sorted]]]))
        assert np.array_equal(got, exp), (r, int(perm[i_sorted]))
    ref_c = oracle.counts(parts, params)
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    for got, key in zip(g["counts"], ("grav", "gather", "sym")):
        assert np.array_equal(got[inv], ref_c[key]), key


@pytest.mark.parametrize("kk,inside", [((1289220, 989691, 0), False), ((848717, 414813, 1322568), True)])
@pytest.mark.parametrize("sym", [1, 0])
def test_production_gravity_count_predicate_edges(kk, inside, sym):
    """The two fp32-predicate edge pairs of tests/test_oracle_pins.py through the GPU's gravity
    kernels (Newton-3 pipelined and i-centric): s32 == rcut2 exactly (out) and the pair whose
    fma sequence stays below rcut2 while its exact s rounds to it (in)."""
    from gen.configs import make_params, quantise

    box = [16.0] * 3
    params = make_params(box, symmetric=sym)
    q = 16.0 * 2.0**-23
    pos = quantise(np.array([[1.0, 1, 1], 1.0 + np.asarray(kk, np.float64) * q]), box)
    parts = dict(x=pos[:, 0].copy(), y=pos[:, 1].copy(), z=pos[:, 2].copy(),
                 vx=np.zeros(2, np.float32), vy=np.zeros(2, np.float32), vz=np.zeros(2, np.float32),
                 m=np.ones(2, np.float32), species=np.zeros(2, np.uint8), id=np.arange(2, dtype=np.int64),
                 H=np.zeros(2, np.float32), u=np.zeros(2, np.float32))
    g = run_gpu(parts, params, hydro=False)
    assert g["cnt_in"][0].tolist() == ([1, 1] if inside else [0, 0])
    assert oracle.counts(parts, params)["grav"].tolist() == g["cnt_in"][0].tolist()


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_gravity_pipe_configurations_counts_and_forces(cfg):
    """The pipelined Newton-3 kernel's three launch configurations (grav_kernel 0-2: shared
    leaf capacity 20 / 32 / 16, 5 / 4 / 6 CTAs per SM — the L2 fallback past the staged
    leaves included) give the oracle's counts and forces on c2z."""
    from crk_testutil import norm_err

    parts, params = cached_config("c2z")
    params["grav_kernel"] = cfg
    g = run_gpu(parts, params, hydro=False)
    ref_c = oracle.counts(parts, params)
    assert np.array_equal(g["cnt_in"][0], ref_c["grav"])
    ref = oracle.gravity(parts, params)
    a = np.stack([g["in"][k] for k in ("ax", "ay", "az")], 1)
    assert norm_err(a, ref["a"], ref["S"]) <= 1e-4
