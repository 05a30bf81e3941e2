"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2310_16122_b200) never imports it and shares no code with it.

The arithmetic lives in oracle.c (plain C, fp64, OpenMP), which follows
SURVEY.md §8(c) O1-O9 step by step; this module only marshals numpy arrays
and computes the dependency closure of sampled targets (which particles'
intermediates a sampled output needs).  See DESIGN.md §2 for the readings
of the paper (arxiv 2310.16122) that the oracle implements.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# tools/mutation_check.py points this at a deliberately mutated build of oracle.c to show that
# the pins in tests/ catch each mutation; nothing else sets it
_LIB_OVERRIDE = os.environ.get("CRK_ORACLE_LIB")

CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc, fp64, no FP contraction so the fp32 predicate is exact)."""
    if _LIB_OVERRIDE:
        return _LIB_OVERRIDE
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class Params(C.Structure):
    _fields_ = [
        ("box", C.c_double * 3),
        ("rcut2", C.c_float), ("eps2", C.c_float), ("poly", C.c_float * 6), ("G", C.c_float),
        ("gamma", C.c_float), ("av_cl", C.c_float), ("av_cq", C.c_float), ("av_eps2", C.c_float),
        ("leaf_max_i", C.c_int32), ("leaf_max_j", C.c_int32),
        ("leaf_max_gas_i", C.c_int32), ("leaf_max_gas_j", C.c_int32),
        ("cell_side", C.c_double),
    ]


def params_struct(p: dict) -> Params:
    s = Params()
    s.box[:] = p["box"]
    for k in ("rcut2", "eps2", "G", "gamma", "av_cl", "av_cq", "av_eps2", "cell_side"):
        setattr(s, k, p[k])
    s.poly[:] = p["poly"]
    for k in ("leaf_max_i", "leaf_max_j", "leaf_max_gas_i", "leaf_max_gas_j"):
        setattr(s, k, p[k])
    return s


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_leaves.restype = C.c_int64
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f32(parts, k):
    return np.ascontiguousarray(parts[k], dtype=np.float32)


def _targets(parts, targets):
    n = parts["x"].shape[0]
    if targets is None:
        return np.arange(n, dtype=np.int64)
    return np.ascontiguousarray(targets, dtype=np.int64)


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_threads(n: int) -> None:
    """OpenMP threads of the following oracle calls."""
    lib().orc_set_threads(C.c_int(int(n)))


# ----------------------------------------------------------------- O3 / O4
def sort_order(parts, params):
    n = parts["x"].shape[0]
    order = np.empty(n, np.int64)
    keys = np.empty(n, np.uint64)
    cellm = np.empty(n, np.uint64)
    rc = lib().orc_sort(C.c_int64(n), _p(_f32(parts, "x")), _p(_f32(parts, "y")), _p(_f32(parts, "z")),
                        _p(np.ascontiguousarray(parts["id"], np.int64)), C.byref(params_struct(params)),
                        _p(order), _p(keys), _p(cellm))
    if rc != 0:
        raise ValueError("bad parameters (box / cell side must be powers of two)")
    return order, keys, cellm


def leaves(parts, params, order, cellm, kind):
    """kind 0 grav-i, 1 grav-j, 2 gas-i, 3 gas-j (see oracle.c)."""
    n = parts["x"].shape[0]
    ps = params_struct(params)
    args = [C.c_int64(n), _p(order), _p(cellm), _p(_f32(parts, "x")), _p(_f32(parts, "y")),
            _p(_f32(parts, "z")), _p(np.ascontiguousarray(parts["species"], np.uint8)),
            _p(_f32(parts, "H")), C.byref(ps), C.c_int(kind)]
    nl = lib().orc_leaves(*args, None, None, None, None, None)
    first = np.empty(nl, np.int64)
    count = np.empty(nl, np.int32)
    bbox = np.empty((nl, 6), np.float32)
    maxh2 = np.zeros(nl, np.float32)
    cell = np.empty(nl, np.uint64)
    lib().orc_leaves(*args, _p(first), _p(count), _p(bbox), _p(maxh2), _p(cell))
    return dict(first=first, count=count, bbox=bbox, maxh2=maxh2, cell=cell)


def list_rows(la, lb, params, mode, rows=None):
    """CSR rows of the leaf-pair list for i-leaves `rows` (default all).  mode 0: gravity
    (cut2 = rcut2); mode 1: hydro (cut2 = max of the two leaves' max H^2)."""
    if rows is None:
        rows = np.arange(la["count"].shape[0], dtype=np.int64)
    rows = np.ascontiguousarray(rows, np.int64)
    ps = params_struct(params)
    nr = rows.shape[0]
    nb = lb["count"].shape[0]
    lens = np.empty(nr, np.int64)
    ba, bb = np.ascontiguousarray(la["bbox"]), np.ascontiguousarray(lb["bbox"])
    ma, mb = np.ascontiguousarray(la["maxh2"]), np.ascontiguousarray(lb["maxh2"])
    lib().orc_list_rows(C.c_int64(nr), _p(rows), _p(ba), _p(ma), C.c_int64(nb), _p(bb), _p(mb),
                        C.byref(ps), C.c_int(mode), _p(lens), None, None, None)
    off = np.zeros(nr + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    col = np.empty(off[-1], np.int32)
    sh = np.empty(off[-1], np.int8)
    lib().orc_list_rows(C.c_int64(nr), _p(rows), _p(ba), _p(ma), C.c_int64(nb), _p(bb), _p(mb),
                        C.byref(ps), C.c_int(mode), _p(lens), _p(off), _p(col), _p(sh))
    return off, col, sh


# ----------------------------------------------------------------- O2 counts
def counts(parts, params, targets=None, brute=False):
    t = _targets(parts, targets)
    nt = t.shape[0]
    cg, ch, cs = (np.empty(nt, np.int32) for _ in range(3))
    lib().orc_counts(C.c_int64(parts["x"].shape[0]), _p(_f32(parts, "x")), _p(_f32(parts, "y")),
                     _p(_f32(parts, "z")), _p(np.ascontiguousarray(parts["species"], np.uint8)),
                     _p(_f32(parts, "H")), C.byref(params_struct(params)), C.c_int64(nt), _p(t),
                     _p(cg), _p(ch), _p(cs), C.c_int(int(brute)))
    return dict(grav=cg, gather=ch, sym=cs)


# ----------------------------------------------------------------- passes
def gravity(parts, params, targets=None, dt=0.0, brute=False):
    t = _targets(parts, targets)
    nt = t.shape[0]
    a = np.empty((nt, 3))
    S = np.empty(nt)
    v = np.empty((nt, 3))
    lib().orc_gravity(C.c_int64(parts["x"].shape[0]), _p(_f32(parts, "x")), _p(_f32(parts, "y")),
                      _p(_f32(parts, "z")), _p(_f32(parts, "m")), _p(_f32(parts, "vx")),
                      _p(_f32(parts, "vy")), _p(_f32(parts, "vz")), C.byref(params_struct(params)),
                      C.c_double(dt), C.c_int64(nt), _p(t), _p(a), _p(S), _p(v), C.c_int(int(brute)))
    return dict(a=a, S=S, v=v)


def geometry(parts, params, targets, brute=False):
    t = _targets(parts, targets)
    V = np.empty(t.shape[0])
    lib().orc_geometry(C.c_int64(parts["x"].shape[0]), _p(_f32(parts, "x")), _p(_f32(parts, "y")),
                       _p(_f32(parts, "z")), _p(np.ascontiguousarray(parts["species"], np.uint8)),
                       _p(_f32(parts, "H")), C.byref(params_struct(params)), C.c_int64(t.shape[0]),
                       _p(t), _p(V), C.c_int(int(brute)))
    return V


def corrections(parts, params, V, targets, brute=False):
    t = _targets(parts, targets)
    nt = t.shape[0]
    A = np.empty(nt)
    B = np.empty((nt, 3))
    dA = np.empty((nt, 3))
    dB = np.empty((nt, 9))
    lib().orc_corrections(C.c_int64(parts["x"].shape[0]), _p(_f32(parts, "x")), _p(_f32(parts, "y")),
                          _p(_f32(parts, "z")), _p(np.ascontiguousarray(parts["species"], np.uint8)),
                          _p(_f32(parts, "H")), _p(np.ascontiguousarray(V, np.float64)),
                          C.byref(params_struct(params)), C.c_int64(nt), _p(t), _p(A), _p(B), _p(dA),
                          _p(dB), C.c_int(int(brute)))
    return dict(A=A, B=B, dA=dA, dB=dB)


def _d(a, n, w=None):
    a = np.ascontiguousarray(a, np.float64)
    return a


def extras(parts, params, V, A, B, dA, dB, targets, v=None, brute=False):
    """v: optional (n,3) fp32 velocities overriding parts' (e.g. after a kick)."""
    t = _targets(parts, targets)
    nt = t.shape[0]
    rho, P, cs = np.empty(nt), np.empty(nt), np.empty(nt)
    dv = np.empty((nt, 9))
    vx, vy, vz = (_f32(parts, k) for k in ("vx", "vy", "vz")) if v is None else \
        (np.ascontiguousarray(v[:, k], np.float32) for k in range(3))
    lib().orc_extras(C.c_int64(parts["x"].shape[0]), _p(_f32(parts, "x")), _p(_f32(parts, "y")),
                     _p(_f32(parts, "z")), _p(np.ascontiguousarray(parts["species"], np.uint8)),
                     _p(_f32(parts, "H")), _p(_f32(parts, "m")), _p(vx), _p(vy), _p(vz),
                     _p(_f32(parts, "u")), _p(_d(V, 1)), _p(_d(A, 1)), _p(_d(B, 3)), _p(_d(dA, 3)),
                     _p(_d(dB, 9)), C.byref(params_struct(params)), C.c_int64(nt), _p(t), _p(rho),
                     _p(P), _p(cs), _p(dv), C.c_int(int(brute)))
    return dict(rho=rho, P=P, cs=cs, dv=dv)


def accel(parts, params, V, A, B, dA, dB, rho, P, cs, dv, targets, dt=0.0, v=None, brute=False):
    t = _targets(parts, targets)
    nt = t.shape[0]
    a = np.empty((nt, 3))
    du, Sa, Sdu, uo = np.empty(nt), np.empty(nt), np.empty(nt), np.empty(nt)
    vo = np.empty((nt, 3))
    vx, vy, vz = (_f32(parts, k) for k in ("vx", "vy", "vz")) if v is None else \
        (np.ascontiguousarray(v[:, k], np.float32) for k in range(3))
    lib().orc_accel(C.c_int64(parts["x"].shape[0]), _p(_f32(parts, "x")), _p(_f32(parts, "y")),
                    _p(_f32(parts, "z")), _p(np.ascontiguousarray(parts["species"], np.uint8)),
                    _p(_f32(parts, "H")), _p(_f32(parts, "m")), _p(vx), _p(vy), _p(vz),
                    _p(_f32(parts, "u")), _p(_d(V, 1)), _p(_d(A, 1)), _p(_d(B, 3)), _p(_d(dA, 3)),
                    _p(_d(dB, 9)), _p(_d(rho, 1)), _p(_d(P, 1)), _p(_d(cs, 1)), _p(_d(dv, 9)),
                    C.byref(params_struct(params)), C.c_double(dt), C.c_int64(nt), _p(t), _p(a),
                    _p(du), _p(Sa), _p(Sdu), _p(vo), _p(uo), C.c_int(int(brute)))
    return dict(a=a, dudt=du, Sa=Sa, Sdu=Sdu, v=vo, u=uo)


def kernel(r, H):
    W, g = C.c_double(), C.c_double()
    lib().orc_kernel(C.c_double(r), C.c_double(H), C.byref(W), C.byref(g))
    return W.value, g.value


def corrected_kernel(A, B, dA, dB, d, H):
    B, dA, dB, d = (np.ascontiguousarray(v, np.float64) for v in (B, dA, dB, d))
    WR = C.c_double()
    g = np.empty(3)
    lib().orc_corrected_kernel(C.c_double(A), _p(B), _p(dA), _p(dB), _p(d), C.c_double(H),
                               C.byref(WR), _p(g))
    return WR.value, g


def neighbour_sets(parts, params, targets, pred):
    """Sorted neighbour index arrays of each target; pred 1 = gather incl. self, 2 = sym."""
    t = _targets(parts, targets)
    nt = t.shape[0]
    args = [C.c_int64(parts["x"].shape[0]), _p(_f32(parts, "x")), _p(_f32(parts, "y")),
            _p(_f32(parts, "z")), _p(np.ascontiguousarray(parts["species"], np.uint8)),
            _p(_f32(parts, "H")), C.byref(params_struct(params)), C.c_int(pred), C.c_int64(nt), _p(t)]
    lens = np.empty(nt, np.int64)
    lib().orc_neighbour_sets(*args, _p(lens), None, None)
    off = np.zeros(nt + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    out = np.empty(off[-1], np.int64)
    lib().orc_neighbour_sets(*args, _p(lens), _p(off), _p(out))
    return off, out


# ----------------------------------------------------------------- the substep chain
def substep(parts, params, targets=None, dt_grav=0.0, dt_hydro=0.0, brute=False, hydro=True,
            grav_targets=None):
    """Run the short-range substep in the GPU call order (gravity kick, geometry,
    corrections, extras, accel/du) and return every output for the requested gas
    `targets` (default: every particle).  For sampled targets the intermediates are
    computed only on the dependency closure; other entries stay NaN."""
    n = parts["x"].shape[0]
    gas = np.ascontiguousarray(parts["species"]) == 1
    full = targets is None
    out = {}
    gt = np.arange(n, dtype=np.int64) if (full and grav_targets is None) else grav_targets
    if gt is not None:
        g = gravity(parts, params, gt, dt_grav, brute)
        out["grav_targets"] = np.asarray(gt)
        out.update(grav_a=g["a"], grav_S=g["S"], grav_v=g["v"])
    if not hydro:
        return out
    if full:
        T3 = np.nonzero(gas)[0].astype(np.int64)
        T2 = T1 = T3
    else:
        T3 = np.unique(np.asarray(targets, np.int64))
        assert gas[T3].all(), "hydro targets must be gas"
        off, nb = neighbour_sets(parts, params, T3, 2)
        T2 = np.unique(np.concatenate([T3, nb]))
        off, nb = neighbour_sets(parts, params, T2, 1)
        T1 = np.unique(np.concatenate([T2, nb]))
    v = None
    if dt_grav != 0.0:
        g1 = gravity(parts, params, T1, dt_grav, brute)
        v = np.stack([parts["vx"], parts["vy"], parts["vz"]], 1).astype(np.float64)
        v[T1] = g1["v"]
        v = v.astype(np.float32)
    nan = lambda *s: np.full((n,) + s, np.nan)  # noqa: E731
    V = nan()
    V[T1] = geometry(parts, params, T1, brute)
    cr = corrections(parts, params, V, T2, brute)
    A, B, dA, dB = nan(), nan(3), nan(3), nan(9)
    A[T2], B[T2], dA[T2], dB[T2] = cr["A"], cr["B"], cr["dA"], cr["dB"]
    ex = extras(parts, params, V, A, B, dA, dB, T2, v=v, brute=brute)
    rho, P, cs, dv = nan(), nan(), nan(), nan(9)
    rho[T2], P[T2], cs[T2], dv[T2] = ex["rho"], ex["P"], ex["cs"], ex["dv"]
    ac = accel(parts, params, V, A, B, dA, dB, rho, P, cs, dv, T3, dt_hydro, v=v, brute=brute)
    out.update(targets=T3, V=V[T3], A=A[T3], B=B[T3], dA=dA[T3], dB=dB[T3], rho=rho[T3], P=P[T3],
               cs=cs[T3], dv=dv[T3], a=ac["a"], dudt=ac["dudt"], Sa=ac["Sa"], Sdu=ac["Sdu"],
               v=ac["v"], u=ac["u"])
    return out


# ----------------------------------------------------------------- sub-cycle (NEXT-2)
def courant_dt(species, H, cs, a, ah, params, c_cfl=0.25, c_acc=0.25):
    """dt = min_i of C_acc sqrt(eps/|a_i|) (a + a_h for gas) and, for gas, C_cfl H_i / c_i (fp64)."""
    n = species.shape[0]
    f = lambda v: np.ascontiguousarray(v, np.float32)  # noqa: E731
    lib().orc_courant.restype = C.c_double
    return float(lib().orc_courant(C.c_int64(n), _p(np.ascontiguousarray(species, np.uint8)), _p(f(H)), _p(f(cs)),
                                   _p(f(a[:, 0])), _p(f(a[:, 1])), _p(f(a[:, 2])), _p(f(ah[:, 0])), _p(f(ah[:, 1])),
                                   _p(f(ah[:, 2])), C.c_double(params["eps2"]), C.c_double(c_cfl),
                                   C.c_double(c_acc)))


def kick(species, v, u, a, ah, dudt, dt):
    """v += dt (a + a_h for gas), u += dt du/dt (gas), one fp32 fma each; returns new (v, u)."""
    n = species.shape[0]
    f = lambda x: np.ascontiguousarray(x, np.float32).copy()  # noqa: E731
    vx, vy, vz, uu = f(v[:, 0]), f(v[:, 1]), f(v[:, 2]), f(u)
    lib().orc_kick(C.c_int64(n), _p(np.ascontiguousarray(species, np.uint8)), C.c_float(dt),
                   _p(f(a[:, 0])), _p(f(a[:, 1])), _p(f(a[:, 2])), _p(f(ah[:, 0])), _p(f(ah[:, 1])), _p(f(ah[:, 2])),
                   _p(f(dudt)), _p(vx), _p(vy), _p(vz), _p(uu))
    return np.stack([vx, vy, vz], 1), uu


def drift(x, v, box, dt):
    """x' = fl32(x + dt v) on the q lattice, wrapped (fp32, bit-exact specification)."""
    n = x.shape[0]
    xs = [np.ascontiguousarray(x[:, a], np.float32).copy() for a in range(3)]
    vs = [np.ascontiguousarray(v[:, a], np.float32) for a in range(3)]
    b = (C.c_double * 3)(*box)
    lib().orc_drift(C.c_int64(n), b, C.c_float(dt), _p(xs[0]), _p(xs[1]), _p(xs[2]), _p(vs[0]), _p(vs[1]), _p(vs[2]))
    return np.stack(xs, 1)


def knn_h(parts, params, targets, k=64, factor=1.01):
    """H' = fl32(factor * sqrt(k-th smallest s32 to another gas particle)) and whether that
    neighbour lies inside the current H (brute force over every gas particle)."""
    t = _targets(parts, targets)
    Hn = np.empty(t.shape[0], np.float32)
    conv = np.empty(t.shape[0], np.int32)
    b = (C.c_double * 3)(*params["box"])
    lib().orc_knn_h(C.c_int64(parts["x"].shape[0]), _p(_f32(parts, "x")), _p(_f32(parts, "y")), _p(_f32(parts, "z")),
                    _p(np.ascontiguousarray(parts["species"], np.uint8)), _p(_f32(parts, "H")), b,
                    C.c_int64(t.shape[0]), _p(t), C.c_int(k), C.c_float(factor), _p(Hn), _p(conv))
    return Hn, conv.astype(bool)


# ----------------------------------------------------------------- long-range PM (NEXT-3)
def pm_accel(x, y, z, m, box, n_grid, r_s, G=1.0):
    """Long-range particle-mesh acceleration in fp64 (DESIGN.md §2 "Long-range PM"):
    cloud-in-cell deposit (cell centres at (i + 1/2) dx), rho_k by a real FFT,
    phi_k = -4 pi G exp(-k^2 r_s^2) / k^2 rho_k (zero mode dropped), a_k = -i k phi_k with
    the Nyquist component of each derivative zeroed, inverse FFTs, cloud-in-cell
    interpolation.  Plain numpy steps in the order of the method."""
    L = float(box[0])
    ng = int(n_grid)
    dx = L / ng
    pos = np.stack([np.asarray(x, np.float64), np.asarray(y, np.float64), np.asarray(z, np.float64)], 1) / dx - 0.5
    base = np.floor(pos)
    f = pos - base
    i0 = np.mod(base.astype(np.int64), ng)
    i1 = np.mod(i0 + 1, ng)
    w = [(1.0 - f[:, a], f[:, a]) for a in range(3)]
    idx = [(i0[:, a], i1[:, a]) for a in range(3)]
    rho = np.zeros((ng, ng, ng))
    mm = np.asarray(m, np.float64) / dx ** 3
    for a in range(2):
        for b in range(2):
            for c in range(2):
                np.add.at(rho, (idx[0][a], idx[1][b], idx[2][c]), mm * w[0][a] * w[1][b] * w[2][c])
    rk = np.fft.rfftn(rho)
    kf = 2.0 * np.pi / L * np.fft.fftfreq(ng, 1.0 / ng)
    kh = 2.0 * np.pi / L * np.arange(ng // 2 + 1)
    KX, KY, KZ = np.meshgrid(kf, kf, kh, indexing="ij")
    k2 = KX ** 2 + KY ** 2 + KZ ** 2
    with np.errstate(divide="ignore", invalid="ignore"):
        g = np.where(k2 > 0, -4.0 * np.pi * G * np.exp(-k2 * r_s ** 2) / k2, 0.0)
    phi = g * rk
    nyq = ng // 2
    D = [KX.copy(), KY.copy(), KZ.copy()]
    D[0][nyq, :, :] = 0.0
    D[1][:, nyq, :] = 0.0
    D[2][:, :, nyq] = 0.0
    out = []
    for a in range(3):
        grid = np.fft.irfftn(-1j * D[a] * phi, s=(ng, ng, ng), axes=(0, 1, 2))
        acc = np.zeros(pos.shape[0])
        for ia in range(2):
            for ib in range(2):
                for ic in range(2):
                    acc += w[0][ia] * w[1][ib] * w[2][ic] * grid[idx[0][ia], idx[1][ib], idx[2][ic]]
        out.append(acc)
    return np.stack(out, 1)
