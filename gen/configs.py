"""Input recipe (SURVEY.md §8(d) "Concrete synthetic inputs").

Every array is generated from a numpy Generator seeded with
``seed = 16122 + 100*config + variant`` and returned in a *shuffled* order
(ids stay attached), so that the solver's sort is exercised.

Units: the mean inter-particle spacing per species is 1 (grid units, Δ);
the box is n_a per axis.  Positions are quantised to q = L_max * 2^-23
(our reading) so that every periodic difference of two
positions is exact in fp32.

Species: 0 = dark matter (gravity only), 1 = gas (gravity + CRK-SPH)
(§3.1 "separate particle species").
"""
from __future__ import annotations

import math
import numpy as np

F_B = 0.157  # baryon fraction: m_gas = f_b, m_dm = 1 - f_b (mean density 1 per Δ^3)


# --------------------------------------------------------------------------- params
def fit_grid_poly(rc: float, eps2: float, rs_over: float = 4.5, order: int = 5):
    """Degree-5 polynomial in s = r^2 standing in for HACC's fitted grid force
    (PAPER.md:646 ``HACC_CUDA_POLY_ORDER=5``; the paper does not print it, so
    this is SURVEY.md §8(c) O5's reading): least squares on s in [0, rc^2] to
    the Gaussian-split long-range force per unit separation
    [erf(r/2r_s) - r/(r_s sqrt(pi)) exp(-r^2/4r_s^2)] / r^3, r_s = rc/rs_over,
    constrained so that P5(rc^2) = (rc^2 + eps2)^-3/2 (short-range force
    vanishes at the cutoff).  Returns fp32-rounded coefficients c_0..c_5.
    This is an *input* of the method, generated offline like HACC's."""
    from scipy.special import erf

    rs = rc / rs_over
    s = np.linspace(0.0, rc * rc, 2001)
    r = np.sqrt(s)
    f = np.empty_like(s)
    small = r < 1e-3
    rr = r[~small]
    f[~small] = (erf(rr / (2 * rs)) - rr / (rs * math.sqrt(math.pi)) * np.exp(-rr * rr / (4 * rs * rs))) / rr**3
    f[small] = 1.0 / (6.0 * math.sqrt(math.pi) * rs**3)  # r -> 0 limit
    return fit_poly_samples(s, f, rc, eps2, order)


def fit_poly_samples(s, f, rc: float, eps2: float, order: int = 5):
    """Least-squares polynomial in s to samples f(s) of a long-range force per unit
    separation, constrained to P(rc^2) = (rc^2 + eps2)^-3/2 (KKT system).  With samples of
    the force a particle-mesh solver actually produces (``PM.force_profile``) this is how
    HACC derives its grid-force polynomial; fp32 coefficients."""
    s = np.asarray(s, np.float64)
    f = np.asarray(f, np.float64)
    V = np.vander(s, order + 1, increasing=True)
    cvec = (rc * rc) ** np.arange(order + 1)
    target = (rc * rc + eps2) ** -1.5
    n = order + 1
    K = np.zeros((n + 1, n + 1))
    K[:n, :n] = 2 * V.T @ V
    K[:n, n] = cvec
    K[n, :n] = cvec
    rhs = np.concatenate([2 * V.T @ f, [target]])
    sol = np.linalg.solve(K, rhs)
    return np.asarray(sol[:n], dtype=np.float32)


def make_params(box, rc=3.1, eps2=0.01, G=1.0, gamma=5.0 / 3.0, av_cl=2.0, av_cq=1.0,
                av_eps2=0.01, leaf_max_i=128, leaf_max_j=8, leaf_max_gas_i=64,
                leaf_max_gas_j=8, cell_side=4.0, poly=None, symmetric=1, skin=0.0, grav_kernel=0,
                hydro_kernel=0, nbr_cap=0):
    """Parameter set (SURVEY.md §8(b) crk_params; defaults §8(c) O5-O9, §8(d))."""
    box = [float(b) for b in box]
    if poly is None:
        poly = fit_grid_poly(rc, eps2)
    return dict(
        box=box,
        rcut2=float(np.float32(rc * rc)),
        eps2=float(np.float32(eps2)),
        poly=[float(c) for c in np.asarray(poly, dtype=np.float32)],
        G=float(np.float32(G)),
        gamma=float(np.float32(gamma)),
        av_cl=float(np.float32(av_cl)),
        av_cq=float(np.float32(av_cq)),
        av_eps2=float(np.float32(av_eps2)),
        leaf_max_i=int(leaf_max_i),
        leaf_max_j=int(leaf_max_j),
        leaf_max_gas_i=int(leaf_max_gas_i),
        leaf_max_gas_j=int(leaf_max_gas_j),
        cell_side=float(cell_side),
        symmetric=int(symmetric),  # kernel variant bitmask (solver option, not physics)
        skin=float(np.float32(skin)),  # list skin (solver option, not physics)
        # kernel variants and neighbour-list capacity (solver options, include/crksr.h)
        grav_kernel=int(grav_kernel), hydro_kernel=int(hydro_kernel), nbr_cap=int(nbr_cap),
    )


# --------------------------------------------------------------------------- helpers
def quantise(pos: np.ndarray, box) -> np.ndarray:
    """Round to multiples of q = L_max 2^-23 and wrap into [0, L_a) (O1)."""
    box = np.asarray(box, dtype=np.float64)
    q = float(box.max()) * 2.0**-23
    k = np.floor(pos / q + 0.5).astype(np.int64)
    kmax = np.round(box / q).astype(np.int64)
    k = np.mod(k, kmax)
    return (k.astype(np.float64) * q).astype(np.float32)


def zeldovich_psi(shape, amp, rng):
    """Gaussian random displacement ψ = ∇φ on the lattice, P(k) ∝ k^-1 exp(-(k/k_Nyq)^2),
    scaled to rms |ψ| = amp.  Returns (nx,ny,nz,3) float64."""
    nx, ny, nz = shape
    if amp == 0.0:
        return np.zeros((nx, ny, nz, 3))
    kx = np.fft.fftfreq(nx) * 2 * np.pi
    ky = np.fft.fftfreq(ny) * 2 * np.pi
    kz = np.fft.rfftfreq(nz) * 2 * np.pi
    KX, KY, KZ = np.meshgrid(kx, ky, kz, indexing="ij")
    k2 = KX**2 + KY**2 + KZ**2
    knyq = np.pi
    with np.errstate(divide="ignore", invalid="ignore"):
        amp_k = np.where(k2 > 0, np.sqrt(k2) ** -0.5 * np.exp(-0.5 * k2 / knyq**2), 0.0)
    delta = np.fft.rfftn(rng.standard_normal((nx, ny, nz)))
    delta *= amp_k
    psi = np.empty((nx, ny, nz, 3))
    with np.errstate(divide="ignore", invalid="ignore"):
        for a, K in enumerate((KX, KY, KZ)):
            comp = np.where(k2 > 0, 1j * K / k2, 0.0) * delta
            psi[..., a] = np.fft.irfftn(comp, s=(nx, ny, nz), axes=(0, 1, 2))
    rms = math.sqrt(float(np.mean(np.sum(psi**2, axis=-1))))
    return psi * (amp / rms)


def smoothing_lengths(gas_pos: np.ndarray, box, k: int = 64, factor: float = 1.01):
    """H_i = 1.01 x distance to the 64th-nearest gas neighbour (fp64, periodic),
    SURVEY.md §8(c) O6 reading; gives ~66 gather neighbours."""
    from scipy.spatial import cKDTree

    if gas_pos.shape[0] <= k:
        raise ValueError("need more than %d gas particles" % k)
    tree = cKDTree(gas_pos.astype(np.float64), boxsize=np.asarray(box, dtype=np.float64))
    d, _ = tree.query(gas_pos.astype(np.float64), k=k + 1, workers=-1)
    return (factor * d[:, k]).astype(np.float32)


def _assemble(box, pos_dm, pos_gas, v_dm, v_gas, rng, shuffle=True):
    n_dm, n_gas = pos_dm.shape[0], pos_gas.shape[0]
    pos = np.concatenate([pos_dm, pos_gas])
    vel = np.concatenate([v_dm, v_gas]).astype(np.float32)
    species = np.concatenate([np.zeros(n_dm, np.uint8), np.ones(n_gas, np.uint8)])
    m = np.where(species == 1, np.float32(F_B), np.float32(1.0 - F_B)).astype(np.float32)
    pos = quantise(pos, box)
    H = np.zeros(n_dm + n_gas, np.float32)
    H[n_dm:] = smoothing_lengths(pos[n_dm:], box)
    u = np.zeros(n_dm + n_gas, np.float32)
    u[n_dm:] = (1.0 * np.exp(0.1 * rng.standard_normal(n_gas))).astype(np.float32)
    ids = np.arange(n_dm + n_gas, dtype=np.int64)
    order = rng.permutation(n_dm + n_gas) if shuffle else np.arange(n_dm + n_gas)
    return dict(
        x=np.ascontiguousarray(pos[order, 0]), y=np.ascontiguousarray(pos[order, 1]),
        z=np.ascontiguousarray(pos[order, 2]),
        vx=np.ascontiguousarray(vel[order, 0]), vy=np.ascontiguousarray(vel[order, 1]),
        vz=np.ascontiguousarray(vel[order, 2]),
        m=m[order], species=species[order], id=ids[order], H=H[order], u=u[order],
    )


def make_lattice(shape, amp, seed, shuffle=True, vel_scale=1.0):
    """Two interleaved lattices: DM at (i,j,k)+1/4+ψ, gas at +3/4+ψ, v = ψ (f=1)."""
    rng = np.random.default_rng(seed)
    nx, ny, nz = shape
    box = [float(nx), float(ny), float(nz)]
    psi = zeldovich_psi(shape, amp, rng)
    grid = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1)
    grid = grid.reshape(-1, 3).astype(np.float64)
    psi = psi.reshape(-1, 3)
    pos_dm = grid + 0.25 + psi
    pos_gas = grid + 0.75 + psi
    v = psi * vel_scale
    return box, _assemble(box, pos_dm, pos_gas, v, v, rng, shuffle)


def make_clustered(n, seed, n_halos=512, frac_halo=0.5, rho_cap=200.0, mmin=256, mmax=65536,
                   shuffle=True):
    """50% of each species in Plummer halos (centres uniform,
    dN/dM ∝ M^-2 on [mmin, mmax], scale radius a = (3M/(4π ρ_cap))^(1/3),
    truncated at 8a), the rest a uniform Poisson background."""
    rng = np.random.default_rng(seed)
    L = float(n)
    box = [L, L, L]
    n_sp = n**3
    n_halo_tot = int(round(frac_halo * n_sp))
    # inverse-CDF sample of dN/dM ∝ M^-2
    uu = rng.random(n_halos)
    M = 1.0 / (1.0 / mmin - uu * (1.0 / mmin - 1.0 / mmax))
    counts = np.floor(M / M.sum() * n_halo_tot).astype(np.int64)
    counts[np.argsort(-M)[: n_halo_tot - counts.sum()]] += 1
    centres = rng.random((n_halos, 3)) * L
    a = (3.0 * counts / (4.0 * np.pi * rho_cap)) ** (1.0 / 3.0)

    def species_positions():
        parts = [rng.random((n_sp - n_halo_tot, 3)) * L]
        vels = [np.zeros((n_sp - n_halo_tot, 3))]
        for c, cnt, ah in zip(centres, counts, a):
            # Plummer radius by inverse CDF, truncated at 8a
            umax = (64.0 / 65.0) ** 1.5
            uv = rng.random(cnt) * umax
            r = ah / np.sqrt(uv ** (-2.0 / 3.0) - 1.0)
            d = rng.standard_normal((cnt, 3))
            d /= np.linalg.norm(d, axis=1, keepdims=True)
            parts.append(c + d * r[:, None])
            sig = 0.3 * math.sqrt(cnt / 2048.0)
            vels.append(rng.standard_normal((cnt, 3)) * sig)
        return np.mod(np.concatenate(parts), L), np.concatenate(vels)

    pos_dm, v_dm = species_positions()
    pos_gas, v_gas = species_positions()
    return box, _assemble(box, pos_dm, pos_gas, v_dm, v_gas, rng, shuffle)


# --------------------------------------------------------------------------- configs
CONFIGS = {
    # name: (config number, variant, kind, n, amplitude)
    "c1": (1, 0, "lattice", 16, 0.05),
    "c2u": (2, 0, "lattice", 64, 0.0),
    "c2z": (2, 1, "lattice", 64, 0.1),
    "c3": (3, 0, "clustered", 128, None),
    "c4": (4, 0, "lattice", 256, 0.1),
}


def make_config(name: str, shuffle: bool = True, **param_overrides):
    """Return (parts, params) for a named config (BASELINE.json configs 1-4;
    config 5 per GPU is config 4's 2x256^3 size)."""
    if name.startswith("lat"):
        # custom small lattice: "lat:nx,ny,nz:amp:seed"
        _, dims, amp, seed = name.split(":")
        shape = tuple(int(t) for t in dims.split(","))
        box, parts = make_lattice(shape, float(amp), int(seed), shuffle)
        return parts, make_params(box, **param_overrides)
    cfg, var, kind, n, amp = CONFIGS[name]
    seed = 16122 + 100 * cfg + var
    if kind == "lattice":
        box, parts = make_lattice((n, n, n), amp, seed, shuffle)
    else:
        box, parts = make_clustered(n, seed, shuffle=shuffle)
    return parts, make_params(box, **param_overrides)
