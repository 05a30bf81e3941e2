"""Sub-cycle steps: time-step limit, kick, drift on the q lattice.

CPU: the oracle's kick / drift / time step against closed forms and invariants.
GPU (-m gpu): crk_courant_dt, crk_kick, crk_drift against the oracle on the same sorted
arrays (drift and kick bit-exact: both are specified in fp32; the time step within fp32
rounding of the per-particle terms), and a two-step kick-drift-kick against the oracle's.
"""
import math

import numpy as np
import pytest

import oracle
from crk_testutil import cached_config

Q_BITS = 23


def _q(box):
    return math.ldexp(max(box), -Q_BITS)


# ----------------------------------------------------------------- CPU pins
def test_drift_stays_on_lattice_and_wraps():
    box = [16.0, 8.0, 8.0]
    q = _q(box)
    rng = np.random.default_rng(5)
    n = 4000
    x = np.floor(rng.random((n, 3)) * np.array(box) / q) * q
    v = rng.normal(0, 3.0, (n, 3)).astype(np.float32)
    y = oracle.drift(x.astype(np.float32), v, box, 0.37)
    assert np.all(np.mod(y.astype(np.float64), q) == 0.0)  # multiples of q (O1)
    for a in range(3):
        assert np.all((y[:, a] >= 0) & (y[:, a] < box[a]))
    # closed form away from rounding: |fl(x + dt v) - (x + dt v)| <= ulp, then <= q/2 to the lattice
    exact = np.mod(x + 0.37 * v.astype(np.float64), np.array(box))
    d = np.abs(y - exact)
    d = np.minimum(d, np.array(box) - d)
    assert np.all(d <= q / 2 + 1e-6 * np.array(box))


def test_drift_exact_cases():
    box = [8.0, 8.0, 8.0]
    q = _q(box)
    x = np.array([[1.0, 7.5, 0.25]], np.float32)
    v = np.array([[0.0, 2.0, -1.0]], np.float32)
    y = oracle.drift(x, v, box, 0.5)  # dt v = (0, 1, -0.5): exact, with wraps on y and z
    assert np.array_equal(y, np.array([[1.0, 0.5, 7.75]], np.float32))
    back = oracle.drift(y, v, box, -0.5)
    assert np.array_equal(back, x)
    # a step of a quarter quantum rounds back to the lattice point (ties to even: 0.5 q -> 0)
    y = oracle.drift(x, np.array([[q / 4, q / 2, 0.0]], np.float32), box, 1.0)
    assert y[0, 0] == x[0, 0] and y[0, 1] == x[0, 1]
    # to the NEAREST lattice point, in both directions: +3q/4 goes up a quantum, -q/4 stays
    # (rounding toward zero would give x and z - q)
    y = oracle.drift(x, np.array([[0.75 * q, 0.0, -0.25 * q]], np.float32), box, 1.0)
    assert np.array_equal(y, np.array([[1.0 + q, 7.5, 0.25]], np.float32))


def test_kick_closed_form():
    sp = np.array([0, 1], np.uint8)
    v = np.array([[1.0, 0.0, -1.0], [0.5, 0.25, 0.0]], np.float32)
    u = np.array([0.0, 2.0], np.float32)
    a = np.array([[2.0, -4.0, 0.0], [1.0, 1.0, 1.0]], np.float32)
    ah = np.array([[100.0, 100.0, 100.0], [1.0, -1.0, 3.0]], np.float32)  # ignored for DM
    dudt = np.array([9.0, -2.0], np.float32)
    v2, u2 = oracle.kick(sp, v, u, a, ah, dudt, 0.5)
    assert np.array_equal(v2, np.array([[2.0, -2.0, -1.0], [1.5, 0.25, 2.0]], np.float32))
    assert np.array_equal(u2, np.array([0.0, 1.0], np.float32))


def test_courant_closed_forms():
    params = {"eps2": 0.01}
    n = 10
    sp = np.array([1] * 5 + [0] * 5, np.uint8)
    H = np.full(n, 2.0, np.float32)
    cs = np.full(n, 4.0, np.float32)
    z = np.zeros((n, 3), np.float32)
    # no accelerations: the sound-crossing limit C_cfl H / c
    assert oracle.courant_dt(sp, H, cs, z, z, params, 0.3, 0.25) == pytest.approx(0.3 * 2.0 / 4.0, rel=1e-15)
    # a uniform acceleration 9 on the dark matter only: C_acc sqrt(eps / 9) (eps = 0.1) is smaller
    a = z.copy()
    a[5:, 0] = 9.0
    want = min(0.3 * 0.5, 0.25 * math.sqrt(0.1 / 9.0))
    assert oracle.courant_dt(sp, H, cs, a, z, params, 0.3, 0.25) == pytest.approx(want, rel=1e-15)
    # gas: gravity and hydro accelerations add (3-4-0 + 0-0-12 -> |a| = 13)
    a2, ah = z.copy(), z.copy()
    a2[0] = (3.0, 4.0, 0.0)
    ah[0] = (0.0, 0.0, 12.0)
    want = min(0.3 * 0.5, 0.25 * math.sqrt(0.1 / 13.0))
    assert oracle.courant_dt(sp, H, cs, a2, ah, params, 0.3, 0.25) == pytest.approx(want, rel=1e-15)


# ----------------------------------------------------------------- GPU parity
def _gpu_state(name):
    import torch
    from paper_2310_16122_b200 import Particles, Solver

    parts, params = cached_config(name)
    p = Particles.from_host(parts, "cuda")
    s = Solver(params, 0)
    s.substep(p)
    torch.cuda.synchronize()
    return parts, params, p, s


def _host(p, keys):
    return {k: getattr(p, k).cpu().numpy() for k in keys}


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2z"])
def test_gpu_courant_kick_drift(name):
    parts, params, p, s = _gpu_state(name)
    h = _host(p, ["x", "y", "z", "vx", "vy", "vz", "u", "H", "species", "cs", "ax", "ay", "az", "ahx", "ahy",
                  "ahz", "dudt"])
    a = np.stack([h["ax"], h["ay"], h["az"]], 1)
    ah = np.stack([h["ahx"], h["ahy"], h["ahz"]], 1)
    dt = s.courant_dt(p, 0.25, 0.3)
    ref = oracle.courant_dt(h["species"], h["H"], h["cs"], a, ah, params, 0.25, 0.3)
    assert abs(dt - ref) <= 1e-6 * ref
    # kick: bit-exact (one fp32 fma per component on both sides)
    s.kick(p, 0.5 * dt)
    v0 = np.stack([h["vx"], h["vy"], h["vz"]], 1)
    vk, uk = oracle.kick(h["species"], v0, h["u"], a, ah, h["dudt"], np.float32(0.5 * dt))
    g = _host(p, ["vx", "vy", "vz", "u"])
    assert np.array_equal(np.stack([g["vx"], g["vy"], g["vz"]], 1), vk)
    assert np.array_equal(g["u"], uk)
    # drift: bit-exact, on the q lattice
    s.drift(p, dt)
    xd = oracle.drift(np.stack([h["x"], h["y"], h["z"]], 1), vk, params["box"], np.float32(dt))
    g = _host(p, ["x", "y", "z"])
    assert np.array_equal(np.stack([g["x"], g["y"], g["z"]], 1), xd)
    s.close()


@pytest.mark.gpu
def test_gpu_drift_requires_rebuild():
    from paper_2310_16122_b200.binding import CrkError

    parts, params, p, s = _gpu_state("c1")
    s.drift(p, 0.0)
    with pytest.raises(CrkError):
        s.gravity_kick(p)
    s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("skin", [0.0, 0.3])
def test_gpu_kdk_two_steps_matches_oracle(skin):
    """Two kick-drift-kick sub-cycles on c1 against the oracle's sequence (forces from
    oracle.substep, the GPU's time steps): positions within a few q, velocities and u
    within the force tolerance accumulated over the kicks."""
    import torch
    from paper_2310_16122_b200 import Particles, Solver

    parts, params = cached_config("c1")
    params["skin"] = skin  # > 0: the second force evaluation reuses the lists (crk_refresh)
    p = Particles.from_host(parts, "cuda")
    s = Solver(params, 0)
    dts = s.kdk(p, 2, 0.25, 0.3)
    torch.cuda.synchronize()
    h = p.to_host()
    s.close()
    # the oracle's sequence in input order (the GPU sorts in place; compare by id)
    st = {k: parts[k].copy() for k in parts}
    n = st["x"].shape[0]
    gas = st["species"] == 1

    def forces(st):
        ref = oracle.substep(st, params)
        a = ref["grav_a"].astype(np.float32)
        ah = np.zeros((n, 3), np.float32)
        du = np.zeros(n, np.float32)
        ah[ref["targets"]] = ref["a"]
        du[ref["targets"]] = ref["dudt"]
        return a, ah, du

    def do_kick(st, dt, f):
        v, u = oracle.kick(st["species"], np.stack([st["vx"], st["vy"], st["vz"]], 1), st["u"], f[0], f[1], f[2], dt)
        st["vx"], st["vy"], st["vz"], st["u"] = v[:, 0].copy(), v[:, 1].copy(), v[:, 2].copy(), u

    f = forces(st)
    for dt in dts:
        do_kick(st, np.float32(0.5 * dt), f)
        x = oracle.drift(np.stack([st["x"], st["y"], st["z"]], 1), np.stack([st["vx"], st["vy"], st["vz"]], 1),
                         params["box"], np.float32(dt))
        st["x"], st["y"], st["z"] = x[:, 0].copy(), x[:, 1].copy(), x[:, 2].copy()
        f = forces(st)
        do_kick(st, np.float32(0.5 * dt), f)
    pos_of_id = np.empty(n, np.int64)
    pos_of_id[h["id"]] = np.arange(n)
    g = pos_of_id[st["id"]]
    q = _q(params["box"])
    L = np.array(params["box"])
    dx = np.abs(np.stack([h["x"][g], h["y"][g], h["z"][g]], 1) - np.stack([st["x"], st["y"], st["z"]], 1))
    dx = np.minimum(np.mod(dx, L), L - np.mod(dx, L))  # skin drifts leave positions unwrapped
    assert np.max(dx) <= 4 * q
    v_ref = np.stack([st["vx"], st["vy"], st["vz"]], 1).astype(np.float64)
    v_gpu = np.stack([h["vx"][g], h["vy"][g], h["vz"][g]], 1)
    dv0 = np.abs(v_ref - np.stack([parts["vx"], parts["vy"], parts["vz"]], 1)).max()
    assert np.max(np.abs(v_gpu - v_ref)) <= 1e-4 * dv0 + 1e-6 * np.abs(v_ref).max()
    du0 = np.abs(st["u"] - parts["u"]).max()
    assert np.max(np.abs(h["u"][g] - st["u"])) <= 1e-4 * du0 + 1e-6 * np.abs(st["u"]).max()


# ----------------------------------------------------------------- smoothing-length update
def _lattice_gas(n=16):
    from gen.configs import make_params

    g = (np.arange(n) + 0.75).astype(np.float64)
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    N = n ** 3
    parts = dict(x=X.ravel().astype(np.float32), y=Y.ravel().astype(np.float32), z=Z.ravel().astype(np.float32),
                 vx=np.zeros(N, np.float32), vy=np.zeros(N, np.float32), vz=np.zeros(N, np.float32),
                 m=np.ones(N, np.float32), species=np.ones(N, np.uint8), id=np.arange(N, dtype=np.int64),
                 H=np.full(N, 2.6, np.float32), u=np.ones(N, np.float32))
    return parts, make_params([float(n)] * 3)


def test_knn_h_lattice_shells():
    """Unit lattice: shells of 6, 12, 8, 6, 24, 24 points at d^2 = 1..6, so the 64th
    neighbour is on the d^2 = 6 shell (56 closer) and the 6th on the d^2 = 1 shell."""
    parts, params = _lattice_gas()
    t = np.array([0, 123, 4000])
    Hn, conv = oracle.knn_h(parts, params, t, k=64, factor=1.01)
    assert np.all(Hn == np.float32(1.01) * np.sqrt(np.float32(6.0)))
    assert np.all(conv)  # 6 < 2.6^2
    Hn, conv = oracle.knn_h(parts, params, t, k=6, factor=1.0)
    assert np.all(Hn == 1.0)
    Hn, conv = oracle.knn_h(parts, params, t, k=57, factor=1.0)
    assert np.all(Hn == np.sqrt(np.float32(6.0)))
    # a smaller H puts the 64th neighbour outside: not converged
    parts["H"][:] = 2.0
    Hn, conv = oracle.knn_h(parts, params, t, k=64, factor=1.01)
    assert not np.any(conv)


def test_knn_h_matches_numpy_ranking():
    """Random gas: the oracle's k-th distance agrees with an fp64 numpy ranking."""
    from gen.configs import make_params, quantise

    rng = np.random.default_rng(9)
    n, L = 600, 8.0
    pos = quantise(rng.random((n, 3)) * L, [L] * 3)
    parts = dict(x=pos[:, 0].copy(), y=pos[:, 1].copy(), z=pos[:, 2].copy(), species=np.ones(n, np.uint8),
                 H=np.full(n, 1.5, np.float32))
    params = make_params([L] * 3)
    t = np.arange(0, n, 37)
    Hn, _ = oracle.knn_h(parts, params, t, k=20, factor=1.0)
    p = pos.astype(np.float64)
    for q, i in enumerate(t):
        d = p - p[i]
        d -= L * np.round(d / L)
        r = np.sort(np.sqrt((d * d).sum(1)))[1:]  # drop self
        assert abs(float(Hn[q]) - r[19]) <= 2e-6 * r[19]


@pytest.mark.gpu
@pytest.mark.parametrize("name,scale", [("c1", 1.0), ("c1", 0.85), ("c2z", 1.0)])
def test_gpu_update_h(name, scale):
    """crk_update_h after geometry: converged particles bit-exact with the oracle's kNN,
    the unconverged count equal to the oracle's."""
    import torch
    from paper_2310_16122_b200 import Particles, Solver

    parts, params = cached_config(name)
    parts["H"] = (parts["H"] * np.float32(scale)).astype(np.float32)
    p = Particles.from_host(parts, "cuda")
    s = Solver(params, 0)
    s.build_lists(p)
    s.geometry(p)
    Hn, nu = s.update_h(p, 64, 1.01)
    torch.cuda.synchronize()
    h = p.to_host(["perm", "species"])
    Hg = np.empty_like(parts["H"])
    Hg[h["perm"].astype(np.int64)] = Hn.cpu().numpy()
    gas = np.nonzero(parts["species"] == 1)[0]
    t = gas if name == "c1" else np.sort(np.random.default_rng(2).choice(gas, 300, replace=False))
    Hr, conv = oracle.knn_h(parts, params, t, 64, 1.01)
    assert np.array_equal(Hg[t][conv], Hr[conv])
    if name == "c1":
        assert nu == int((~conv).sum())
    s.close()


@pytest.mark.gpu
def test_gpu_adapt_h_converges_to_knn():
    """Starting from H x 0.8 (most 64th neighbours outside H), build -> geometry -> update_h
    iterations converge, and the final H is the oracle's kNN value for every sampled particle."""
    from paper_2310_16122_b200 import Particles, Solver

    parts, params = cached_config("c2z")
    parts["H"] = (parts["H"] * np.float32(0.8)).astype(np.float32)
    p = Particles.from_host(parts, "cuda")
    s = Solver(params, 0)
    it = s.adapt_h(p, 64, 1.01)
    assert 2 <= it <= 4
    h = p.to_host(["perm", "H", "x", "y", "z", "species", "id"])
    s.close()
    gas = np.nonzero(h["species"] == 1)[0]
    t = np.sort(np.random.default_rng(4).choice(gas, 200, replace=False))
    sorted_parts = {k: h[k] for k in ("x", "y", "z", "species", "H")}
    Hr, _ = oracle.knn_h(sorted_parts, params, t, 64, 1.01)
    assert np.array_equal(h["H"][t], Hr)


# ----------------------------------------------------------------- skin lists (list reuse)
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2z"])
def test_gpu_skin_refresh_matches_oracle(name):
    """Lists built with a skin, then drifts totalling < skin/2 and crk_refresh instead of a
    rebuild: counts exact and forces within the bar against the oracle on the drifted
    positions; past skin/2 the refresh refuses and a rebuild restores the passes."""
    import torch
    from paper_2310_16122_b200 import Particles, Solver
    from paper_2310_16122_b200.binding import CrkError
    from crk_testutil import norm_err

    parts, params = cached_config(name)
    params["skin"] = 0.4
    p = Particles.from_host(parts, "cuda")
    s = Solver(params, 0)
    s.substep(p)
    vmag = float(np.sqrt(parts["vx"].astype(np.float64) ** 2 + parts["vy"] ** 2 + parts["vz"] ** 2).max())
    dt = 0.09 / vmag  # each drift moves the fastest particle by 0.09 (skin/2 = 0.2)
    L = np.array(params["box"])

    def passes_and_check():
        s.gravity_kick(p)
        s.geometry(p)
        s.corrections_extras(p)
        s.hydro_accel_dudt(p)
        torch.cuda.synchronize()
        h = p.to_host()
        pos_of_id = np.empty(parts["id"].shape[0], np.int64)
        pos_of_id[parts["id"]] = np.arange(parts["id"].shape[0])
        perm = pos_of_id[h["id"]]  # sorted position -> input index (ids survive every re-sort)
        cur = {k: parts[k].copy() for k in parts}
        for k in ("x", "y", "z"):
            v = np.empty_like(parts[k])
            v[perm] = np.mod(h[k].astype(np.float64), L["xyz".index(k)]).astype(np.float32)
            cur[k] = v
        cg, ch, cs = s.count_pairs(p)
        ref_c = oracle.counts(cur, params)
        for c, want in zip((cg, ch, cs), ("grav", "gather", "sym")):
            got = np.empty(perm.shape[0], np.int32)
            got[perm] = c.cpu().numpy()
            assert np.array_equal(got, ref_c[want]), want
        gas = np.nonzero(cur["species"] == 1)[0]
        t = gas if name == "c1" else np.sort(np.random.default_rng(6).choice(gas, 200, replace=False))
        ref = oracle.substep(cur, params, targets=t, grav_targets=t)
        inv = lambda a: a[np.argsort(perm)]  # noqa: E731  sorted -> input order
        a = np.stack([inv(h["ax"]), inv(h["ay"]), inv(h["az"])], 1)[t]
        assert norm_err(a, ref["grav_a"], ref["grav_S"]) <= 1e-4
        T = ref["targets"]
        ah = np.stack([inv(h["ahx"]), inv(h["ahy"]), inv(h["ahz"])], 1)[T]
        assert norm_err(ah, ref["a"], ref["Sa"]) <= 1e-4
        assert norm_err(inv(h["dudt"])[T], ref["dudt"], ref["Sdu"]) <= 1e-4

    passes_and_check()
    for _ in range(2):  # 2 x 0.09 < 0.2
        s.drift(p, dt)
        s.refresh(p)
        passes_and_check()
    s.drift(p, dt)  # 0.27 >= 0.2: a refresh must refuse
    with pytest.raises(CrkError):
        s.refresh(p)
    s.build_lists(p)
    passes_and_check()
    s.close()
