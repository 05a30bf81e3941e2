"""GPU (sm_100a) vs fp64 oracle parity, through the C-ABI (libcrksr.so).

Bars (north_star, SURVEY.md §8(c) "Tolerance"):
  * sort order, leaves, interaction lists, neighbour counts: bit-exact;
  * gravity acceleration, hydro acceleration, du/dt: max_i |gpu - ref| / S_i <= 1e-4,
    S_i = sum_j |pair contribution| (fp32 vs fp64);
  * intermediates: V, A, rho, P, c relative <= 1e-5; B, grad A, grad B, grad v made
    dimensionless with the particle's H (|dB| H, |d grad A| H / A, |d grad B| H^2,
    |d grad v| H / v_rms) <= 2e-5, 1e-4 for grad B (DESIGN.md §6 derives these from
    fp32 cancellation in the moment sums).
"""
import numpy as np
import pytest

import oracle
from crk_testutil import cached_config, run_gpu, norm_err, rel_err, dimless_err

pytestmark = pytest.mark.gpu

TOL_FORCE = 1e-4


def _oracle_lists(parts, params):
    order, keys, cellm = oracle.sort_order(parts, params)
    ls = [oracle.leaves(parts, params, order, cellm, k) for k in range(4)]
    lists = [oracle.list_rows(ls[0], ls[1], params, 0), oracle.list_rows(ls[2], ls[3], params, 1)]
    return order, ls, lists


def _canon_rows(off, col, sh):
    rows = []
    for a in range(off.shape[0] - 1):
        c = np.asarray(col[off[a]:off[a + 1]], np.int64)
        s = np.asarray(sh[off[a]:off[a + 1]], np.int64)
        o = np.lexsort((s, c))
        rows.append((c[o], s[o]))
    return rows


@pytest.mark.parametrize("name", ["c1", "lat:32,16,16:0.1:3", "c2z"])
def test_sort_leaves_lists_bit_exact(name):
    parts, params = cached_config(name)
    g = run_gpu(parts, params, counts=False, lists=True, hydro=False)
    order, ls, lists = _oracle_lists(parts, params)
    assert np.array_equal(g["perm"], order)
    lv = g["lv"]
    for s in range(4):
        gl = {k: (v.cpu().numpy() if v is not None else None) for k, v in lv["leaves"][s].items()}
        assert np.array_equal(gl["first"], ls[s]["first"]), s
        assert np.array_equal(gl["count"], ls[s]["count"]), s
        assert np.array_equal(gl["bbox"], ls[s]["bbox"]), s
        assert np.array_equal(gl["cell"].astype(np.uint64), ls[s]["cell"]), s
        if s >= 2:
            assert np.array_equal(gl["maxh2"], ls[s]["maxh2"]), s
    for m in range(2):
        off, col, sh = lists[m]
        gv = lv["lists"][m]
        goff = gv["row_off"].cpu().numpy()
        assert np.array_equal(goff, off), m
        rg = _canon_rows(goff, gv["col"].cpu().numpy(), gv["shift"].cpu().numpy())
        ro = _canon_rows(off, col, sh)
        for a, (x, y) in enumerate(zip(rg, ro)):
            assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1]), (m, a)


@pytest.mark.parametrize("name,sym", [("c1", 3), ("c1", 0), ("c1", 4), ("lat:32,16,16:0.1:3", 3), ("c2u", 0),
                                      ("c2z", 3), ("c2z", 0), ("c2z", 5)])
def test_counts_and_full_chain(name, sym):
    parts, params = cached_config(name)
    params["symmetric"] = sym
    g = run_gpu(parts, params)
    ref_c = oracle.counts(parts, params)
    cg, ch, cs = g["cnt_in"]
    assert np.array_equal(cg, ref_c["grav"])
    assert np.array_equal(ch, ref_c["gather"])
    assert np.array_equal(cs, ref_c["sym"])
    ref = oracle.substep(parts, params)
    gi = g["in"]
    a = np.stack([gi["ax"], gi["ay"], gi["az"]], 1)
    assert norm_err(a, ref["grav_a"], ref["grav_S"]) <= TOL_FORCE
    T = ref["targets"]
    assert rel_err(gi["V"][T], ref["V"]) <= 1e-5
    assert rel_err(gi["A"][T], ref["A"]) <= 1e-5
    H = parts["H"][T].astype(np.float64)[:, None]
    assert dimless_err(gi["B"][:, T].T, ref["B"], H) <= 2e-5
    assert dimless_err(gi["dA"][:, T].T, ref["dA"], H / ref["A"][:, None]) <= 2e-5
    assert dimless_err(gi["dB"][:, T].T, ref["dB"], H * H) <= 1e-4
    assert rel_err(gi["rho"][T], ref["rho"]) <= 1e-5
    assert rel_err(gi["P"][T], ref["P"]) <= 1e-5
    assert rel_err(gi["cs"][T], ref["cs"]) <= 1e-5
    vrms = np.sqrt(np.mean(parts["vx"] ** 2 + parts["vy"] ** 2 + parts["vz"] ** 2))
    if vrms > 0:
        assert dimless_err(gi["dv"][:, T].T, ref["dv"], H / vrms) <= 2e-5
    ah = np.stack([gi["ahx"], gi["ahy"], gi["ahz"]], 1)[T]
    assert norm_err(ah, ref["a"], ref["Sa"]) <= TOL_FORCE
    assert norm_err(gi["dudt"][T], ref["dudt"], ref["Sdu"]) <= TOL_FORCE


@pytest.mark.parametrize("sym", [3, 0])
def test_kicks(sym):
    parts, params = cached_config("c1")
    params["symmetric"] = sym
    dtg, dth = 0.05, 0.02
    g = run_gpu(parts, params, dt_grav=dtg, dt_hydro=dth, counts=False)
    ref = oracle.substep(parts, params, dt_grav=dtg, dt_hydro=dth)
    gi = g["in"]
    v = np.stack([gi["vx"], gi["vy"], gi["vz"]], 1)
    dm = np.nonzero(parts["species"] == 0)[0]
    T = ref["targets"]
    # DM: gravity kick only; gas: gravity then hydro kick
    sv = np.abs(np.stack([parts["vx"], parts["vy"], parts["vz"]], 1)).max() * 2e-7
    assert np.all(np.abs(v[dm] - ref["grav_v"][dm]) <= dtg * TOL_FORCE * ref["grav_S"][dm, None] + sv)
    tolg = dth * TOL_FORCE * ref["Sa"][:, None] + dtg * TOL_FORCE * ref["grav_S"][T, None] + sv
    assert np.all(np.abs(v[T] - ref["v"]) <= tolg)
    su = np.abs(parts["u"]).max() * 2e-7
    assert np.all(np.abs(gi["u"][T] - ref["u"]) <= dth * TOL_FORCE * ref["Sdu"] + su)


def _species_subset(parts, keep):
    idx = np.nonzero(keep)[0]
    return {k: v[idx].copy() for k, v in parts.items()}


def test_edge_all_dark_matter_and_all_gas():
    parts, params = cached_config("c1")
    dm = _species_subset(parts, parts["species"] == 0)
    g = run_gpu(dm, params)
    ref = oracle.substep(dm, params, hydro=False)
    a = np.stack([g["in"]["ax"], g["in"]["ay"], g["in"]["az"]], 1)
    assert norm_err(a, ref["grav_a"], ref["grav_S"]) <= TOL_FORCE
    assert np.array_equal(g["cnt_in"][0], oracle.counts(dm, params)["grav"])
    assert not np.any(g["cnt_in"][1]) and not np.any(g["cnt_in"][2])
    gas = _species_subset(parts, parts["species"] == 1)
    g = run_gpu(gas, params)
    ref = oracle.substep(gas, params)
    ah = np.stack([g["in"]["ahx"], g["in"]["ahy"], g["in"]["ahz"]], 1)
    assert norm_err(ah, ref["a"], ref["Sa"]) <= TOL_FORCE
    rc = oracle.counts(gas, params)
    assert np.array_equal(g["cnt_in"][2], rc["sym"])


def test_deterministic_and_resort_idempotent():
    """i-centric mode (symmetric=0) is bit-reproducible; the sort is idempotent."""
    import torch
    from paper_2310_16122_b200 import Particles, Solver

    parts, params = cached_config("lat:32,16,16:0.1:3")
    params["symmetric"] = 0
    p = Particles.from_host(parts, "cuda")
    s = Solver(params, 0)
    s.substep(p)
    first = {k: v.copy() for k, v in p.to_host().items()}
    s.substep(p)  # already sorted input: same order, same results
    second = p.to_host()
    for k in first:
        assert np.array_equal(first[k], second[k]) or k == "perm", k
    assert np.array_equal(second["perm"], np.arange(p.n))
    torch.cuda.synchronize()


def test_call_order_and_errors():
    from paper_2310_16122_b200 import CrkError, Particles, Solver

    parts, params = cached_config("c1")
    p = Particles.from_host(parts, "cuda")
    s = Solver(params, 0)
    with pytest.raises(CrkError) as e:
        s.gravity_kick(p)
    assert e.value.status == -4
    s.build_lists(p)
    with pytest.raises(CrkError) as e:
        s.extras(p)
    assert e.value.status == -4
    s.geometry(p)
    s.corrections(p)
    s.extras(p)
    s.hydro_accel_dudt(p)


# ------------------------------------------------------------------ full sizes, sampled outputs
def _sampled_lists(parts, params, g, rng, n_rows=200):
    """Full-size list parity on sampled rows: the sort order in full, and
    for n_rows random i-leaves of each list the leaf (first, count, bbox) and the whole CSR
    row, bit-exact after the canonical row sort, against oracle.list_rows(rows=...)."""
    order, keys, cellm = oracle.sort_order(parts, params)
    assert np.array_equal(g["perm"], order)
    lv = g["lv"]
    for m, (ki, kj) in enumerate(((0, 1), (2, 3))):
        la = oracle.leaves(parts, params, order, cellm, ki)
        lb = oracle.leaves(parts, params, order, cellm, kj)
        gl = lv["leaves"][ki]
        nA = la["count"].shape[0]
        assert int(gl["first"].shape[0]) == nA and int(lv["leaves"][kj]["first"].shape[0]) == lb["count"].shape[0]
        rows = np.sort(rng.choice(nA, min(n_rows, nA), replace=False))
        rt = __import__("torch").as_tensor(rows, device=gl["first"].device)
        assert np.array_equal(gl["first"][rt].cpu().numpy(), la["first"][rows])
        assert np.array_equal(gl["count"][rt].cpu().numpy(), la["count"][rows])
        assert np.array_equal(gl["bbox"][rt].cpu().numpy(), la["bbox"][rows])
        off, col, sh = oracle.list_rows(la, lb, params, m, rows)
        gv = lv["lists"][m]
        goff = gv["row_off"].cpu().numpy()
        gcol, gsh = gv["col"], gv["shift"]
        for r, a in enumerate(rows):
            b0, b1 = int(goff[a]), int(goff[a + 1])
            got = _canon_rows(np.array([0, b1 - b0]), gcol[b0:b1].cpu().numpy(), gsh[b0:b1].cpu().numpy())[0]
            exp = _canon_rows(np.array([0, off[r + 1] - off[r]]), col[off[r]:off[r + 1]], sh[off[r]:off[r + 1]])[0]
            assert np.array_equal(got[0], exp[0]) and np.array_equal(got[1], exp[1]), (m, int(a))


def _sampled(name, n_samp, seed=5):
    parts, params = cached_config(name)
    rng = np.random.default_rng(seed)
    n = parts["x"].shape[0]
    gas = np.nonzero(parts["species"] == 1)[0]
    tg = np.sort(rng.choice(gas, n_samp, replace=False))
    ta = np.sort(rng.choice(n, n_samp, replace=False))
    g = run_gpu(parts, params, lists=True)
    _sampled_lists(parts, params, g, rng)
    ref = oracle.substep(parts, params, targets=tg, grav_targets=ta)
    rc = oracle.counts(parts, params, targets=np.concatenate([ta, tg]))
    gi = g["in"]
    cg, ch, cs = g["cnt_in"]
    allt = np.concatenate([ta, tg])
    assert np.array_equal(cg[allt], rc["grav"])
    assert np.array_equal(ch[allt], rc["gather"])
    assert np.array_equal(cs[allt], rc["sym"])
    a = np.stack([gi["ax"], gi["ay"], gi["az"]], 1)[ta]
    assert norm_err(a, ref["grav_a"], ref["grav_S"]) <= TOL_FORCE
    T = ref["targets"]
    assert rel_err(gi["V"][T], ref["V"]) <= 1e-5
    ah = np.stack([gi["ahx"], gi["ahy"], gi["ahz"]], 1)[T]
    assert norm_err(ah, ref["a"], ref["Sa"]) <= TOL_FORCE
    assert norm_err(gi["dudt"][T], ref["dudt"], ref["Sdu"]) <= TOL_FORCE
    # whole-array properties at full size: momentum conservation of the hydro force
    m = parts["m"].astype(np.float64)
    ahall = np.stack([gi["ahx"], gi["ahy"], gi["ahz"]], 1).astype(np.float64)
    mom = np.abs((m[:, None] * ahall).sum(0))
    assert np.all(mom <= 1e-4 * (m[:, None] * np.abs(ahall)).sum(0).max())
    return g


@pytest.mark.slow
def test_clustered_config3_sampled():
    _sampled("c3", 600)


@pytest.mark.slow
def test_config4_full_size_sampled():
    _sampled("c4", 300)


# ------------------------------------------------------------------ parameter / input edge cases
@pytest.mark.parametrize("li,lg", [(32, 16), (64, 32), (16, 64)])
def test_leaf_size_variants(li, lg):
    """Other compiled leaf sizes: lists, counts and forces still match the oracle."""
    from gen import make_config

    parts, params = make_config("lat:32,16,16:0.12:9", leaf_max_i=li, leaf_max_gas_i=lg)
    g = run_gpu(parts, params, lists=True)
    order, ls, lists = _oracle_lists(parts, params)
    assert np.array_equal(g["perm"], order)
    for m in range(2):
        off, col, sh = lists[m]
        gv = g["lv"]["lists"][m]
        assert np.array_equal(gv["row_off"].cpu().numpy(), off)
    ref_c = oracle.counts(parts, params)
    assert np.array_equal(g["cnt_in"][0], ref_c["grav"])
    assert np.array_equal(g["cnt_in"][2], ref_c["sym"])
    ref = oracle.substep(parts, params)
    gi = g["in"]
    assert norm_err(np.stack([gi["ax"], gi["ay"], gi["az"]], 1), ref["grav_a"], ref["grav_S"]) <= TOL_FORCE
    T = ref["targets"]
    assert norm_err(np.stack([gi["ahx"], gi["ahy"], gi["ahz"]], 1)[T], ref["a"], ref["Sa"]) <= TOL_FORCE


def test_coincident_particles_and_tiny_input():
    """Distinct particles at identical positions (s = 0 pairs), and a box with very few
    particles per cell: counts exact, results finite and within the bar."""
    parts, params = cached_config("c1")
    parts = {k: v.copy() for k, v in parts.items()}
    # move every 97th particle onto its predecessor's position
    for i in range(1, parts["x"].shape[0], 97):
        for k in "xyz":
            parts[k][i] = parts[k][i - 1]
    for sym in (1, 0):
        params["symmetric"] = sym
        g = run_gpu(parts, params)
        ref_c = oracle.counts(parts, params)
        assert np.array_equal(g["cnt_in"][0], ref_c["grav"])
        assert np.array_equal(g["cnt_in"][1], ref_c["gather"])
        assert np.array_equal(g["cnt_in"][2], ref_c["sym"])
        ref = oracle.substep(parts, params)
        gi = g["in"]
        a = np.stack([gi["ax"], gi["ay"], gi["az"]], 1)
        assert np.all(np.isfinite(a))
        assert norm_err(a, ref["grav_a"], ref["grav_S"]) <= TOL_FORCE
        T = ref["targets"]
        assert norm_err(np.stack([gi["ahx"], gi["ahy"], gi["ahz"]], 1)[T], ref["a"], ref["Sa"]) <= TOL_FORCE
    # tiny: 2x4^3 particles in a 16^3 box (mostly empty cells)
    from gen.configs import make_lattice, make_params
    from crk_testutil import cached_config as _cc  # noqa: F401

    rng = np.random.default_rng(3)
    n = 128
    tiny = {k: v[:0] for k, v in parts.items()}
    pos = (rng.random((n, 3)) * 16.0).astype(np.float64)
    from gen.configs import quantise

    pos = quantise(pos, [16.0] * 3)
    tiny = dict(x=pos[:, 0].copy(), y=pos[:, 1].copy(), z=pos[:, 2].copy(),
                vx=np.zeros(n, np.float32), vy=np.zeros(n, np.float32), vz=np.zeros(n, np.float32),
                m=np.full(n, 0.5, np.float32), species=(np.arange(n) % 2).astype(np.uint8),
                id=np.arange(n, dtype=np.int64), H=np.where(np.arange(n) % 2 == 1, 3.5, 0.0).astype(np.float32),
                u=np.ones(n, np.float32))
    tp = make_params([16.0] * 3)
    g = run_gpu(tiny, tp)
    ref_c = oracle.counts(tiny, tp)
    assert np.array_equal(g["cnt_in"][0], ref_c["grav"]) and np.array_equal(g["cnt_in"][2], ref_c["sym"])
    ref = oracle.substep(tiny, tp)
    gi = g["in"]
    assert norm_err(np.stack([gi["ax"], gi["ay"], gi["az"]], 1), ref["grav_a"], ref["grav_S"]) <= TOL_FORCE


@pytest.mark.slow
def test_clustered_config3_full_chain_sampled_symmetric_modes():
    """Config 3 (clustered, dense cells chunked into many leaves, long rows staged in
    several TMA rounds) with both kernel variants."""
    for sym in (0, 3):
        parts, params = cached_config("c3")
        params["symmetric"] = sym
        rng = np.random.default_rng(11)
        gas = np.nonzero(parts["species"] == 1)[0]
        # bias the sample to the densest particles (smallest H)
        dense = gas[np.argsort(parts["H"][gas])[:2000]]
        tg = np.sort(rng.choice(dense, 150, replace=False))
        g = run_gpu(parts, params, counts=False)
        ref = oracle.substep(parts, params, targets=tg, grav_targets=tg)
        gi = g["in"]
        a = np.stack([gi["ax"], gi["ay"], gi["az"]], 1)[tg]
        assert norm_err(a, ref["grav_a"], ref["grav_S"]) <= TOL_FORCE
        T = ref["targets"]
        assert norm_err(np.stack([gi["ahx"], gi["ahy"], gi["ahz"]], 1)[T], ref["a"], ref["Sa"]) <= TOL_FORCE
        assert norm_err(gi["dudt"][T], ref["dudt"], ref["Sdu"]) <= TOL_FORCE


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("cap", [0, 16, 70, 128])
def test_neighbour_list_capacities(cap, fused):
    """The gas passes read the neighbour lists built by geometry; rows whose lists overflow
    the per-particle capacity run the on-the-fly kernels.  cap 0: lists off; 16: every row
    overflows; 70: a mix (sym counts ~64-80 on c2z); 128: no overflow."""
    parts, params = cached_config("c2z")
    params["symmetric"] = 1
    params["nbr_cap"] = cap if cap > 0 else -1
    g = run_gpu(parts, params, counts=False, fused=fused)
    ref = oracle.substep(parts, params)
    gi = g["in"]
    T = ref["targets"]
    assert rel_err(gi["V"][T], ref["V"]) <= 1e-5
    assert rel_err(gi["A"][T], ref["A"]) <= 1e-5
    H = parts["H"][T].astype(np.float64)[:, None]
    assert dimless_err(gi["dB"][:, T].T, ref["dB"], H * H) <= 1e-4
    assert rel_err(gi["rho"][T], ref["rho"]) <= 1e-5
    vrms = np.sqrt(np.mean(parts["vx"] ** 2 + parts["vy"] ** 2 + parts["vz"] ** 2))
    assert dimless_err(gi["dv"][:, T].T, ref["dv"], H / vrms) <= 2e-5
    ah = np.stack([gi["ahx"], gi["ahy"], gi["ahz"]], 1)[T]
    assert norm_err(ah, ref["a"], ref["Sa"]) <= TOL_FORCE
    assert norm_err(gi["dudt"][T], ref["dudt"], ref["Sdu"]) <= TOL_FORCE


@pytest.mark.parametrize("var", [0, 6, 7, 8])
@pytest.mark.parametrize("name", ["c1", "c2z"])
def test_gravity_symmetric_variants(var, name):
    """Every Newton-3 gravity kernel variant (crk_params.grav_kernel) against the oracle."""
    parts, params = cached_config(name)
    params["symmetric"] = 1
    params["grav_kernel"] = var
    g = run_gpu(parts, params, counts=False, hydro=False)
    ref = oracle.substep(parts, params)
    gi = g["in"]
    a = np.stack([gi["ax"], gi["ay"], gi["az"]], 1)
    assert norm_err(a, ref["grav_a"], ref["grav_S"]) <= TOL_FORCE


@pytest.mark.parametrize("var", [5, 4, 6])
@pytest.mark.parametrize("cap", [72, 128])
def test_accel_symmetric_list_variant(cap, var):
    """Opt-in accel list variants: Newton-3 over the neighbour lists (hydro_kernel 5) and
    8 lanes per i (4, 6), with complete lists and with some rows flagged (fallbacks)."""
    parts, params = cached_config("c2z")
    params["symmetric"] = 1
    params["hydro_kernel"] = var
    params["nbr_cap"] = cap
    g = run_gpu(parts, params, counts=False)
    ref = oracle.substep(parts, params)
    gi = g["in"]
    T = ref["targets"]
    ah = np.stack([gi["ahx"], gi["ahy"], gi["ahz"]], 1)[T]
    assert norm_err(ah, ref["a"], ref["Sa"]) <= TOL_FORCE
    assert norm_err(gi["dudt"][T], ref["dudt"], ref["Sdu"]) <= TOL_FORCE


@pytest.mark.parametrize("name,cap", [("c1", 128), ("c2z", 128), ("c2z", 70)])
def test_corrections_extras_one_walk_variant(name, cap):
    """hydro_kernel 2: corrections and extras from ONE walk of each list, Extras' sums carried as
    moments and combined with the new coefficients in the epilogue (the same sums reordered) —
    every intermediate and the accel/du-dt results within the bars, with complete lists and
    with flagged rows (capacity 70: the on-the-fly fallback)."""
    parts, params = cached_config(name)
    params["hydro_kernel"] = 2
    params["nbr_cap"] = cap
    g = run_gpu(parts, params, counts=False)
    ref = oracle.substep(parts, params)
    gi = g["in"]
    T = ref["targets"]
    H = parts["H"][T].astype(np.float64)[:, None]
    assert rel_err(gi["A"][T], ref["A"]) <= 1e-5
    assert dimless_err(gi["B"][:, T].T, ref["B"], H) <= 2e-5
    assert dimless_err(gi["dA"][:, T].T, ref["dA"], H / ref["A"][:, None]) <= 2e-5
    assert dimless_err(gi["dB"][:, T].T, ref["dB"], H * H) <= 1e-4
    assert rel_err(gi["rho"][T], ref["rho"]) <= 1e-5
    assert rel_err(gi["cs"][T], ref["cs"]) <= 1e-5
    vrms = np.sqrt(np.mean(parts["vx"] ** 2 + parts["vy"] ** 2 + parts["vz"] ** 2))
    assert dimless_err(gi["dv"][:, T].T, ref["dv"], H / vrms) <= 2e-5
    ah = np.stack([gi["ahx"], gi["ahy"], gi["ahz"]], 1)[T]
    assert norm_err(ah, ref["a"], ref["Sa"]) <= TOL_FORCE
    assert norm_err(gi["dudt"][T], ref["dudt"], ref["Sdu"]) <= TOL_FORCE
