"""Shared test helpers: generator cache, GPU runner, oracle comparison."""
import numpy as np

_CACHE = {}


def free_port() -> int:
    """A TCP port on 127.0.0.1 that is free right now (for gloo rendezvous in the tests)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def cached_config(name, **kw):
    """Generator outputs are deterministic; cache them per session."""
    from gen import make_config

    key = (name, tuple(sorted(kw.items())))
    if key not in _CACHE:
        _CACHE[key] = make_config(name, **kw)
    parts, params = _CACHE[key]
    return {k: v.copy() for k, v in parts.items()}, dict(params)


FIELDS_SCALAR = ["ax", "ay", "az", "V", "A", "rho", "P", "cs", "ahx", "ahy", "ahz", "dudt"]
FIELDS_PLANES = {"B": 3, "dA": 3, "dB": 9, "dv": 9}


def run_gpu(parts, params, dt_grav=0.0, dt_hydro=0.0, counts=True, lists=False, hydro=True, fused=True):
    """One substep through the C-ABI; outputs mapped back to INPUT order."""
    import torch
    from paper_2310_16122_b200 import Particles, Solver

    dev = torch.device("cuda", 0)
    p = Particles.from_host(parts, dev)
    s = Solver(params, 0)
    s.substep(p, dt_grav, dt_hydro, hydro=hydro, fused=fused)
    res = {}
    if counts:
        cg, ch, cs = s.count_pairs(p)
        res["cnt"] = (cg.cpu().numpy(), ch.cpu().numpy(), cs.cpu().numpy())
    if lists:
        res["lv"] = s.list_view()
    torch.cuda.synchronize()
    res["launches"] = s.launch_count()
    h = p.to_host()
    perm = h["perm"].astype(np.int64)
    res["perm"] = perm
    res["sorted"] = h
    n = perm.shape[0]
    inv = {}
    for k, v in h.items():
        if k == "perm":
            continue
        if v.ndim == 2:
            o = np.empty_like(v)
            o[:, perm] = v
        else:
            o = np.empty_like(v)
            o[perm] = v
        inv[k] = o
    if counts:
        res["cnt_in"] = tuple(_unperm(c, perm) for c in res["cnt"])
    res["in"] = inv
    s.close()
    assert n == parts["x"].shape[0]
    return res


def _unperm(v, perm):
    o = np.empty_like(v)
    o[perm] = v
    return o


def norm_err(gpu, ref, S):
    """max_i |gpu_i - ref_i| / S_i (SURVEY.md §8(c) tolerance), vector rows allowed."""
    d = np.abs(np.asarray(gpu, np.float64) - np.asarray(ref, np.float64))
    if d.ndim == 2:
        d = np.sqrt((d * d).sum(1))
    S = np.asarray(S, np.float64)
    bad = S <= 0
    if np.any(bad):
        assert np.all(d[bad] <= 1e-30), "nonzero result where the oracle sum is empty"
    return float(np.max(d[~bad] / S[~bad])) if np.any(~bad) else 0.0


def rel_err(gpu, ref):
    g = np.asarray(gpu, np.float64)
    r = np.asarray(ref, np.float64)
    return float(np.max(np.abs(g - r) / np.abs(r)))


def scaled_err(gpu, ref):
    """max |gpu - ref| / max |ref| per component (intermediates without a natural S)."""
    g = np.asarray(gpu, np.float64)
    r = np.asarray(ref, np.float64)
    return float(np.max(np.abs(g - r)) / max(np.max(np.abs(r)), 1e-300))


def dimless_err(gpu, ref, scale):
    """max |gpu - ref| * scale (scale makes the field dimensionless, e.g. H for B)."""
    g = np.asarray(gpu, np.float64)
    r = np.asarray(ref, np.float64)
    return float(np.max(np.abs(g - r) * np.asarray(scale, np.float64)))
