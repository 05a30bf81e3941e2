"""Thin ctypes binding of libcrksr.so (include/crksr.h).

Argument marshalling only: every step of the solver runs in the CUDA kernels of
libcrksr.so.  PyTorch supplies device memory and streams.  There is no CPU
fallback: if the library is missing or no GPU is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcrksr.so")

STATUS = {0: "CRK_OK", -1: "CRK_EINVAL", -2: "CRK_ENOMEM", -3: "CRK_ECUDA", -4: "CRK_ESTATE", -5: "CRK_ECAPACITY"}

# exported symbols declared in include/crksr.h (tests check the .so exports all of them)
EXPORTS = ["crk_create", "crk_destroy", "crk_build_lists", "crk_gravity_kick", "crk_geometry",
           "crk_corrections", "crk_extras", "crk_corrections_extras", "crk_hydro_accel_dudt", "crk_count_pairs",
           "crk_list_view", "crk_launch_count", "crk_status_string", "crk_last_error", "crk_select_cells", "crk_select_gas",
           "crk_pack_particles", "crk_unpack_particles", "crk_pack_gas", "crk_unpack_gas", "crk_courant_dt",
           "crk_kick", "crk_drift", "crk_update_h", "crk_refresh", "crk_pm_create", "crk_pm_destroy",
           "crk_pm_accel", "crk_pm_slab_create", "crk_pm_deposit", "crk_pm_slab_forward", "crk_pm_slab_solve",
           "crk_pm_slab_inverse", "crk_pm_interp", "crk_neighbour_lists",
           "crk_select_cells_dev", "crk_select_gas_dev", "crk_pack_particles_dev", "crk_pack_gas_state",
           "crk_unpack_gas_state", "crk_select_rows", "crk_select_peers_dev", "crk_compact_own",
           "crk_select_gas_multi_dev"]


class CrkError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class CrkParams(C.Structure):
    _fields_ = [
        ("box", C.c_double * 3),
        ("rcut2", C.c_float), ("eps2", C.c_float), ("poly", C.c_float * 6), ("G", C.c_float),
        ("gamma", C.c_float), ("av_cl", C.c_float), ("av_cq", C.c_float), ("av_eps2", C.c_float),
        ("leaf_max_i", C.c_int32), ("leaf_max_j", C.c_int32),
        ("leaf_max_gas_i", C.c_int32), ("leaf_max_gas_j", C.c_int32),
        ("cell_side", C.c_double),
        ("symmetric", C.c_int32),
        ("dom_lo", C.c_int32 * 3), ("dom_hi", C.c_int32 * 3),
        ("skin", C.c_float),
        ("grav_kernel", C.c_int32), ("hydro_kernel", C.c_int32), ("nbr_cap", C.c_int32),
    ]


_PF = ["x", "y", "z", "vx", "vy", "vz", "m", "species", "id", "H", "u", "perm", "ax", "ay", "az", "V", "A", "B",
       "dA", "dB", "rho", "P", "cs", "dv", "ahx", "ahy", "ahz", "dudt"]


class CrkParticles(C.Structure):
    _fields_ = [("n", C.c_int64)] + [(k, C.c_void_p) for k in _PF]


class CrkLists(C.Structure):
    _fields_ = [
        ("n_leaf", C.c_int64 * 4),
        ("leaf_first", C.c_void_p * 4), ("leaf_count", C.c_void_p * 4), ("leaf_bbox", C.c_void_p * 4),
        ("leaf_maxh2", C.c_void_p * 4), ("leaf_cell", C.c_void_p * 4),
        ("n_gas", C.c_int64), ("gas_idx", C.c_void_p),
        ("n_entries", C.c_int64 * 2), ("row_off", C.c_void_p * 2), ("col", C.c_void_p * 2),
        ("shift", C.c_void_p * 2),
    ]


_lib = None


def lib():
    """Load libcrksr.so (fails loudly when it is missing: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.crk_create.argtypes = [C.POINTER(CrkParams), C.c_int, C.POINTER(vp)]
        L.crk_destroy.argtypes = [vp]
        for f in ("crk_build_lists", "crk_geometry", "crk_corrections", "crk_extras", "crk_corrections_extras",
                  "crk_refresh"):
            getattr(L, f).argtypes = [vp, C.POINTER(CrkParticles), vp]
        for f in ("crk_gravity_kick", "crk_hydro_accel_dudt"):
            getattr(L, f).argtypes = [vp, C.POINTER(CrkParticles), C.c_float, vp]
        L.crk_count_pairs.argtypes = [vp, C.POINTER(CrkParticles), vp, vp, vp, vp]
        L.crk_neighbour_lists.argtypes = [vp, C.c_int32, vp, vp, vp]
        L.crk_neighbour_lists.restype = C.c_int
        L.crk_courant_dt.argtypes = [vp, C.POINTER(CrkParticles), C.c_float, C.c_float, vp, vp]
        for f in ("crk_kick", "crk_drift"):
            getattr(L, f).argtypes = [vp, C.POINTER(CrkParticles), C.c_float, vp]
        L.crk_update_h.argtypes = [vp, C.POINTER(CrkParticles), C.c_int32, C.c_float, vp, vp, vp]
        L.crk_select_rows.argtypes = [vp, C.c_int32]
        L.crk_select_rows.restype = C.c_int
        L.crk_pm_create.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_float, C.c_float, C.c_int, C.POINTER(vp)]
        L.crk_pm_destroy.argtypes = [vp]
        L.crk_pm_accel.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp]
        L.crk_pm_slab_create.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_float, C.c_float, C.c_int, C.c_int,
                                         C.c_int, C.POINTER(vp)]
        L.crk_pm_deposit.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, vp]
        for f in ("crk_pm_slab_forward", "crk_pm_slab_solve", "crk_pm_slab_inverse"):
            getattr(L, f).argtypes = [vp, vp, vp, vp]
        L.crk_pm_interp.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp]
        for f in ("crk_pm_create", "crk_pm_destroy", "crk_pm_accel", "crk_pm_slab_create", "crk_pm_deposit",
                  "crk_pm_slab_forward", "crk_pm_slab_solve", "crk_pm_slab_inverse", "crk_pm_interp"):
            getattr(L, f).restype = C.c_int
        L.crk_list_view.argtypes = [vp, C.POINTER(CrkLists)]
        L.crk_launch_count.argtypes = [vp]
        L.crk_launch_count.restype = C.c_int64
        L.crk_status_string.argtypes = [C.c_int]
        L.crk_status_string.restype = C.c_char_p
        L.crk_last_error.argtypes = [vp]
        L.crk_last_error.restype = C.c_char_p
        L.crk_select_cells.argtypes = [vp, vp, vp, vp, vp, C.c_int, C.c_int64, C.c_char_p, C.c_char_p, C.c_char_p,
                                       vp, C.POINTER(C.c_int64), vp]
        L.crk_select_gas.argtypes = [vp, C.c_char_p, C.c_char_p, C.c_char_p, vp, C.POINTER(C.c_int64), vp]
        L.crk_pack_particles.argtypes = [vp, C.POINTER(CrkParticles), vp, C.c_int64, vp, vp]
        L.crk_select_cells_dev.argtypes = [vp, vp, vp, vp, vp, C.c_int, C.c_int64, vp, vp, vp, vp]
        L.crk_select_gas_dev.argtypes = [vp, vp, vp, vp, vp]
        L.crk_select_peers_dev.argtypes = [vp, vp, vp, vp, vp, C.c_int64, vp, C.c_int32, vp, C.c_int64, vp, vp]
        L.crk_compact_own.argtypes = [vp, C.POINTER(CrkParticles), C.c_int64, C.POINTER(CrkParticles), vp]
        L.crk_select_gas_multi_dev.argtypes = [vp, vp, C.c_int32, vp, C.c_int64, vp, vp]
        L.crk_pack_particles_dev.argtypes = [vp, C.POINTER(CrkParticles), vp, vp, C.c_int64, vp, vp]
        L.crk_pack_gas_state.argtypes = [vp, C.POINTER(CrkParticles), vp, C.c_int64, vp, vp]
        L.crk_unpack_gas_state.argtypes = [vp, C.POINTER(CrkParticles), vp, C.c_int64, vp, vp]
        for f in ("crk_select_cells_dev", "crk_select_gas_dev", "crk_pack_particles_dev", "crk_pack_gas_state",
                  "crk_unpack_gas_state", "crk_select_peers_dev", "crk_compact_own",
                  "crk_select_gas_multi_dev"):
            getattr(L, f).restype = C.c_int
        L.crk_unpack_particles.argtypes = [vp, C.POINTER(CrkParticles), C.c_int64, C.c_int64, vp, vp]
        L.crk_pack_gas.argtypes = [vp, C.c_int, vp, C.c_int64, vp, vp]
        L.crk_unpack_gas.argtypes = [vp, C.c_int, vp, C.c_int64, vp, vp]
        for f in ("crk_create", "crk_destroy", "crk_build_lists", "crk_gravity_kick", "crk_geometry",
                  "crk_corrections", "crk_extras", "crk_corrections_extras", "crk_hydro_accel_dudt",
                  "crk_count_pairs", "crk_list_view", "crk_select_cells", "crk_select_gas", "crk_pack_particles", "crk_unpack_particles",
                  "crk_pack_gas", "crk_unpack_gas", "crk_courant_dt", "crk_kick", "crk_drift", "crk_update_h",
                  "crk_refresh"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def params_struct(p: dict) -> CrkParams:
    s = CrkParams()
    s.box[:] = p["box"]
    for k in ("rcut2", "eps2", "G", "gamma", "av_cl", "av_cq", "av_eps2", "cell_side"):
        setattr(s, k, p[k])
    s.poly[:] = p["poly"]
    for k in ("leaf_max_i", "leaf_max_j", "leaf_max_gas_i", "leaf_max_gas_j"):
        setattr(s, k, p[k])
    s.symmetric = int(p.get("symmetric", 1))
    s.dom_lo[:] = list(p.get("dom_lo", (0, 0, 0)))
    s.dom_hi[:] = list(p.get("dom_hi", (0, 0, 0)))
    s.skin = float(p.get("skin", 0.0))
    s.grav_kernel = int(p.get("grav_kernel", 0))
    s.hydro_kernel = int(p.get("hydro_kernel", 0))
    s.nbr_cap = int(p.get("nbr_cap", 0))
    return s


class Particles:
    """Device-resident SoA particle set (torch tensors) plus output buffers."""

    IN_F32 = ("x", "y", "z", "vx", "vy", "vz", "m", "H", "u")
    OUT1 = ("ax", "ay", "az", "V", "A", "rho", "P", "cs", "ahx", "ahy", "ahz", "dudt")

    FORCES = ("ax", "ay", "az", "ahx", "ahy", "ahz", "dudt")

    def __init__(self, n: int, device, outputs=True):
        """outputs: True / "all" = every per-particle output incl. the CRK intermediates (V, A,
        B, grad A, grad B, rho, P, c, grad v); "forces" = only the substep's results (gravity
        and hydro accelerations, du/dt; the library skips the intermediate copies); False = none."""
        self.n = int(n)
        self.device = torch.device(device)
        z = lambda *s, dt=torch.float32: torch.zeros(*s, dtype=dt, device=self.device)  # noqa: E731
        for k in self.IN_F32:
            setattr(self, k, z(self.n))
        self.species = z(self.n, dt=torch.uint8)
        self.id = z(self.n, dt=torch.int64)
        self.perm = z(self.n, dt=torch.int32)
        self.outputs = outputs
        if outputs == "forces":
            for k in self.FORCES:
                setattr(self, k, z(self.n))
        elif outputs:
            for k in self.OUT1:
                setattr(self, k, z(self.n))
            self.B = z(3, self.n)
            self.dA = z(3, self.n)
            self.dB = z(9, self.n)
            self.dv = z(9, self.n)

    @classmethod
    def from_host(cls, parts: dict, device="cuda", outputs=True, pinned=None):
        n = parts["x"].shape[0]
        p = cls(n, device, outputs)
        p.load(parts)
        return p

    def load(self, parts: dict, non_blocking=False):
        """Copy host arrays (numpy or pinned torch) to the device buffers."""
        for k in self.IN_F32 + ("species", "id"):
            src = parts[k]
            if not isinstance(src, torch.Tensor):
                src = torch.from_numpy(src)
            getattr(self, k).copy_(src, non_blocking=non_blocking)

    def struct(self) -> CrkParticles:
        s = CrkParticles()
        s.n = self.n
        for k in _PF:
            t = getattr(self, k, None)
            setattr(s, k, t.data_ptr() if t is not None else None)
        return s

    def to_host(self, keys=None) -> dict:
        """Host copies of the first n entries (the arrays may have a larger capacity)."""
        keys = keys or [k for k in _PF if getattr(self, k, None) is not None]
        out = {}
        for k in keys:
            t = getattr(self, k)
            out[k] = (t[:, : self.n] if t.ndim == 2 else t[: self.n]).cpu().numpy()
        return out


class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3}


def _wrap(ptr, shape, typestr, device):
    if int(shape[0]) == 0 or not ptr:
        dt = {"<i4": torch.int32, "<f4": torch.float32, "|i1": torch.int8, "<u8": torch.int64}[typestr]
        return torch.zeros(shape, dtype=dt, device=device)
    t = torch.as_tensor(_CAI(ptr, shape, typestr), device=device)
    return t.clone()


class Solver:
    """One crk_ctx on one device; methods mirror the C-ABI calls of include/crksr.h."""

    def __init__(self, params: dict, device=0):
        self.params = dict(params)
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self._ps = params_struct(params)
        h = C.c_void_p()
        idx = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self._check(lib().crk_create(C.byref(self._ps), idx, C.byref(h)), None)
        self.ctx = h

    def _check(self, st, ctx):
        if st != 0:
            msg = lib().crk_last_error(ctx).decode() if ctx is not None else ""
            raise CrkError(st, msg)

    def close(self):
        if getattr(self, "ctx", None):
            lib().crk_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stream(stream):
        s = stream if stream is not None else torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)

    def _call(self, fn, parts, *args, stream=None):
        ps = parts.struct()
        self._check(fn(self.ctx, C.byref(ps), *args, self._stream(stream)), self.ctx)

    def build_lists(self, parts, stream=None):
        self._call(lib().crk_build_lists, parts, stream=stream)

    def gravity_kick(self, parts, dt=0.0, stream=None):
        self._call(lib().crk_gravity_kick, parts, C.c_float(dt), stream=stream)

    def geometry(self, parts, stream=None):
        self._call(lib().crk_geometry, parts, stream=stream)

    def corrections(self, parts, stream=None):
        self._call(lib().crk_corrections, parts, stream=stream)

    def extras(self, parts, stream=None):
        self._call(lib().crk_extras, parts, stream=stream)

    def corrections_extras(self, parts, stream=None):
        """a5 + a6 fused (crk_corrections_extras): the same results as corrections() then extras()."""
        self._call(lib().crk_corrections_extras, parts, stream=stream)

    def hydro_accel_dudt(self, parts, dt=0.0, stream=None):
        self._call(lib().crk_hydro_accel_dudt, parts, C.c_float(dt), stream=stream)

    ROWS_ALL, ROWS_INTERIOR, ROWS_GHOST = 0, 1, 2

    def select_rows(self, which: int):
        """crk_select_rows: the row subset of the next corrections / extras / accel calls (0 all,
        1 rows whose neighbour rows hold no ghost, 2 the others)."""
        self._check(lib().crk_select_rows(self.ctx, C.c_int32(which)), self.ctx)

    def substep(self, parts, dt_grav=0.0, dt_hydro=0.0, stream=None, hydro=True, fused=True, side_stream=None,
                build=True):
        """The whole short-range substep: a1-a8 in call order.  With
        `side_stream`, gravity (a3) runs there concurrently with geometry (a4) and is joined
        before corrections/extras (which read the kicked v).  build=False reuses refreshed skin
        lists (crk_refresh)."""
        if build:
            self.build_lists(parts, stream)
        if side_stream is not None and hydro:
            main = stream if stream is not None else torch.cuda.current_stream()
            side_stream.wait_stream(main)
            self.gravity_kick(parts, dt_grav, side_stream)
            self.geometry(parts, main)
            main.wait_stream(side_stream)
        else:
            self.gravity_kick(parts, dt_grav, stream)
            if hydro:
                self.geometry(parts, stream)
        if hydro:
            if fused:
                self.corrections_extras(parts, stream)
            else:
                self.corrections(parts, stream)
                self.extras(parts, stream)
            self.hydro_accel_dudt(parts, dt_hydro, stream)

    # ---- sub-cycle ----
    def courant_dt(self, parts, c_cfl=0.25, c_acc=0.25, stream=None):
        """min over particles of the Courant / acceleration limits (crk_courant_dt); syncs."""
        out = torch.empty(1, dtype=torch.float32, device=parts.device)
        self._call(lib().crk_courant_dt, parts, C.c_float(c_cfl), C.c_float(c_acc), C.c_void_p(out.data_ptr()),
                   stream=stream)
        return float(out.item())

    def kick(self, parts, dt, stream=None):
        self._call(lib().crk_kick, parts, C.c_float(dt), stream=stream)

    def drift(self, parts, dt, stream=None):
        self._call(lib().crk_drift, parts, C.c_float(dt), stream=stream)

    def refresh(self, parts, stream=None):
        """Renew the position-dependent data of the skin lists (crk_refresh); syncs."""
        self._call(lib().crk_refresh, parts, stream=stream)

    def update_h(self, parts, k_ngb=64, factor=1.01, stream=None):
        """H' from the k-th nearest gas neighbour among the lists (crk_update_h), after
        geometry.  Returns (H' as a device tensor in sorted order, number unconverged); syncs."""
        H_out = parts.H.clone()
        nu = torch.zeros(1, dtype=torch.int32, device=parts.device)
        self._call(lib().crk_update_h, parts, C.c_int32(k_ngb), C.c_float(factor), C.c_void_p(H_out.data_ptr()),
                   C.c_void_p(nu.data_ptr()), stream=stream)
        return H_out, int(nu.item())

    def adapt_h(self, parts, k_ngb=64, factor=1.01, max_iter=8, stream=None):
        """Iterate build -> geometry -> update_h until every gas particle's k-th neighbour
        lies inside its H (then H = factor x the k-th neighbour distance exactly).  Returns
        the number of iterations."""
        for it in range(1, max_iter + 1):
            self.build_lists(parts, stream)
            self.geometry(parts, stream)
            H_new, nu = self.update_h(parts, k_ngb, factor, stream)
            parts.H.copy_(H_new)
            if nu == 0:
                return it
        raise RuntimeError(f"H did not converge in {max_iter} iterations")

    def kdk(self, parts, n_steps, c_cfl=0.25, c_acc=0.25, stream=None):
        """Kick-drift-kick leapfrog over n_steps sub-cycles, each with the time step of
        crk_courant_dt: forces at x_n, kick dt/2, drift dt, forces at x_{n+1} (the
        velocity-dependent hydro terms see v_{n+1/2}), kick dt/2.  With a list skin
        (params["skin"] > 0) the forces after a drift reuse the lists through crk_refresh
        while the displacement bound allows, else rebuild.  Needs the force outputs (ax..,
        ahx.., dudt).  Returns the time steps taken."""
        self.substep(parts, stream=stream)
        dts = []
        for _ in range(n_steps):
            dt = self.courant_dt(parts, c_cfl, c_acc, stream)
            self.kick(parts, 0.5 * dt, stream)
            self.drift(parts, dt, stream)
            rebuild = True
            if self.params.get("skin", 0.0) > 0.0:
                try:
                    self.refresh(parts, stream)
                    rebuild = False
                except CrkError:
                    pass
            self.substep(parts, stream=stream, build=rebuild)
            self.kick(parts, 0.5 * dt, stream)
            dts.append(dt)
        return dts

    def count_pairs(self, parts, stream=None):
        n = parts.n
        cg = torch.zeros(n, dtype=torch.int32, device=parts.device)
        ch = torch.zeros_like(cg)
        cs = torch.zeros_like(cg)
        ps = parts.struct()
        self._check(lib().crk_count_pairs(self.ctx, C.byref(ps), C.c_void_p(cg.data_ptr()),
                                          C.c_void_p(ch.data_ptr()), C.c_void_p(cs.data_ptr()),
                                          self._stream(stream)), self.ctx)
        return cg, ch, cs

    def neighbour_lists(self, parts, cap_out=160, stream=None):
        """The geometry-built gas neighbour lists (crk_neighbour_lists), decoded to sorted
        positions: (count int32[n] (-1: incomplete list), nbr int32[n, cap_out]) device tensors."""
        cnt = torch.zeros(parts.n, dtype=torch.int32, device=parts.device)
        nbr = torch.full((parts.n, cap_out), -1, dtype=torch.int32, device=parts.device)
        self._check(lib().crk_neighbour_lists(self.ctx, int(cap_out), C.c_void_p(cnt.data_ptr()),
                                              C.c_void_p(nbr.data_ptr()), self._stream(stream)), self.ctx)
        return cnt, nbr

    # ---- ghost exchange (a9) ----
    @staticmethod
    def _mask(m):
        return np.ascontiguousarray(m, dtype=np.uint8).tobytes()

    def select_cells(self, parts, masks, gas_only=False, n=None, stream=None):
        """Indices (device int32) of parts[:n] in the masked cells (masks: 3 uint8 arrays)."""
        n = parts.n if n is None else n
        out = torch.empty(max(n, 1), dtype=torch.int32, device=parts.device)
        cnt = C.c_int64()
        mx, my, mz = (self._mask(m) for m in masks)
        self._check(lib().crk_select_cells(self.ctx, C.c_void_p(parts.x.data_ptr()), C.c_void_p(parts.y.data_ptr()),
                                           C.c_void_p(parts.z.data_ptr()), C.c_void_p(parts.species.data_ptr()),
                                           int(gas_only), n, mx, my, mz, C.c_void_p(out.data_ptr()), C.byref(cnt),
                                           self._stream(stream)), self.ctx)
        return out[: cnt.value]

    def select_gas(self, masks, device, stream=None, n_gas=None):
        out = torch.empty(max(int(n_gas or 1), 1), dtype=torch.int32, device=device)
        cnt = C.c_int64()
        mx, my, mz = (self._mask(m) for m in masks)
        self._check(lib().crk_select_gas(self.ctx, mx, my, mz, C.c_void_p(out.data_ptr()), C.byref(cnt),
                                         self._stream(stream)), self.ctx)
        return out[: cnt.value]

    def select_cells_dev(self, parts, dmask, idx_out, count_dev, n, gas_only=False, stream=None):
        """Indices of parts[:n] in the masked cells into idx_out, the count into count_dev
        (device int32 scalar); dmask: device uint8 (x, y, z masks concatenated); no host sync."""
        self._check(lib().crk_select_cells_dev(self.ctx, C.c_void_p(parts.x.data_ptr()), C.c_void_p(parts.y.data_ptr()),
                                               C.c_void_p(parts.z.data_ptr()), C.c_void_p(parts.species.data_ptr()),
                                               int(gas_only), int(n), C.c_void_p(dmask.data_ptr()),
                                               C.c_void_p(idx_out.data_ptr()), C.c_void_p(count_dev.data_ptr()),
                                               self._stream(stream)), self.ctx)

    def select_peers_dev(self, parts, n, dmasks, idx_out, counts_dev, stream=None):
        """R1 selection of every peer in one pass: dmasks (npeers, ncx + ncy + ncz) uint8 device,
        idx_out (npeers, >= n) int32 device, counts_dev (npeers, 2) int32 device = (all, gas)
        per peer; no host sync (crk_select_peers_dev)."""
        npeers = int(dmasks.shape[0])
        self._check(lib().crk_select_peers_dev(self.ctx, C.c_void_p(parts.x.data_ptr()), C.c_void_p(parts.y.data_ptr()),
                                               C.c_void_p(parts.z.data_ptr()), C.c_void_p(parts.species.data_ptr()),
                                               int(n), C.c_void_p(dmasks.data_ptr()), npeers,
                                               C.c_void_p(idx_out.data_ptr()), int(idx_out.stride(0)),
                                               C.c_void_p(counts_dev.data_ptr()), self._stream(stream)), self.ctx)

    def compact_own(self, src, n_total, n_own, dst, stream=None):
        """dst[:n_own] = the rows of the sorted local set src[:n_total] whose perm < n_own, in
        sorted order (crk_compact_own)."""
        ps, pd = src.struct(), dst.struct()
        ps.n = int(n_total)
        self._check(lib().crk_compact_own(self.ctx, C.byref(ps), int(n_own), C.byref(pd), self._stream(stream)),
                    self.ctx)

    def select_gas_multi_dev(self, dmasks, idx_out, counts_dev, stream=None):
        """crk_select_gas_dev for every row of dmasks (nsets, ncx + ncy + ncz) at once: ascending
        gas ranks of set k in idx_out[k] (nsets, >= n_gas), its size in counts_dev[k]."""
        self._check(lib().crk_select_gas_multi_dev(self.ctx, C.c_void_p(dmasks.data_ptr()), int(dmasks.shape[0]),
                                                   C.c_void_p(idx_out.data_ptr()), int(idx_out.stride(0)),
                                                   C.c_void_p(counts_dev.data_ptr()), self._stream(stream)), self.ctx)

    def select_gas_dev(self, dmask, idx_out, count_dev, stream=None):
        self._check(lib().crk_select_gas_dev(self.ctx, C.c_void_p(dmask.data_ptr()), C.c_void_p(idx_out.data_ptr()),
                                             C.c_void_p(count_dev.data_ptr()), self._stream(stream)), self.ctx)

    def pack_particles_dev(self, parts, idx, count_dev, out, stream=None):
        """R1 records of the first min(count, capacity) selected particles into out (cap, 12) f32."""
        ps = parts.struct()
        self._check(lib().crk_pack_particles_dev(self.ctx, C.byref(ps), C.c_void_p(idx.data_ptr()),
                                                 C.c_void_p(count_dev.data_ptr()), int(out.shape[0]),
                                                 C.c_void_p(out.data_ptr()), self._stream(stream)), self.ctx)

    def pack_particles(self, parts, idx, stream=None):
        out = torch.empty((idx.numel(), 12), dtype=torch.float32, device=parts.device)
        ps = parts.struct()
        self._check(lib().crk_pack_particles(self.ctx, C.byref(ps), C.c_void_p(idx.data_ptr()), idx.numel(),
                                             C.c_void_p(out.data_ptr()), self._stream(stream)), self.ctx)
        return out

    def unpack_particles(self, parts, offset, buf, stream=None):
        ps = parts.struct()
        self._check(lib().crk_unpack_particles(self.ctx, C.byref(ps), int(offset), buf.shape[0],
                                               C.c_void_p(buf.data_ptr()), self._stream(stream)), self.ctx)

    def pack_gas(self, what, idx, stream=None):
        w = 1 if what == 0 else 36
        out = torch.empty((idx.numel(), w), dtype=torch.float32, device=idx.device)
        self._check(lib().crk_pack_gas(self.ctx, int(what), C.c_void_p(idx.data_ptr()), idx.numel(),
                                       C.c_void_p(out.data_ptr()), self._stream(stream)), self.ctx)
        return out

    def pack_gas_state(self, parts, idx, stream=None):
        """R2 records (V, vx, vy, vz) of the gas ranks idx (crk_pack_gas_state)."""
        out = torch.empty((idx.numel(), 4), dtype=torch.float32, device=idx.device)
        ps = parts.struct()
        self._check(lib().crk_pack_gas_state(self.ctx, C.byref(ps), C.c_void_p(idx.data_ptr()), idx.numel(),
                                             C.c_void_p(out.data_ptr()), self._stream(stream)), self.ctx)
        return out

    def unpack_gas_state(self, parts, idx, buf, stream=None):
        ps = parts.struct()
        self._check(lib().crk_unpack_gas_state(self.ctx, C.byref(ps), C.c_void_p(idx.data_ptr()), idx.numel(),
                                               C.c_void_p(buf.data_ptr()), self._stream(stream)), self.ctx)

    def unpack_gas(self, what, idx, buf, stream=None):
        self._check(lib().crk_unpack_gas(self.ctx, int(what), C.c_void_p(idx.data_ptr()), idx.numel(),
                                         C.c_void_p(buf.data_ptr()), self._stream(stream)), self.ctx)

    def launch_count(self) -> int:
        return int(lib().crk_launch_count(self.ctx))

    def list_view(self) -> dict:
        """Copies of the leaves and lists (device tensors)."""
        lv = CrkLists()
        self._check(lib().crk_list_view(self.ctx, C.byref(lv)), self.ctx)
        torch.cuda.synchronize(self.device)
        d = self.device
        out = {"leaves": [], "lists": []}
        for s in range(4):
            nl = lv.n_leaf[s]
            out["leaves"].append(dict(
                first=_wrap(lv.leaf_first[s], (nl,), "<i4", d),
                count=_wrap(lv.leaf_count[s], (nl,), "<i4", d),
                bbox=_wrap(lv.leaf_bbox[s], (nl, 6), "<f4", d),
                maxh2=_wrap(lv.leaf_maxh2[s], (nl,), "<f4", d) if s >= 2 else None,
                cell=_wrap(lv.leaf_cell[s], (nl,), "<u8", d),
            ))
        out["gas_idx"] = _wrap(lv.gas_idx, (lv.n_gas,), "<i4", d)
        for m in range(2):
            na = lv.n_leaf[0 if m == 0 else 2]
            ne = lv.n_entries[m]
            out["lists"].append(dict(
                row_off=_wrap(lv.row_off[m], (na + 1,), "<i4", d),
                col=_wrap(lv.col[m], (ne,), "<i4", d),
                shift=_wrap(lv.shift[m], (ne,), "|i1", d),
            ))
        return out


class PM:
    """Long-range particle-mesh gravity (crk_pm_*): CIC + cuFFT + Gaussian-filtered Poisson."""

    def __init__(self, n_grid: int, box, r_s: float, G: float = 1.0, device=0):
        b = (C.c_double * 3)(*[float(v) for v in box])
        h = C.c_void_p()
        st = lib().crk_pm_create(int(n_grid), b, C.c_float(r_s), C.c_float(G), int(device), C.byref(h))
        if st != 0:
            raise CrkError(st, "crk_pm_create")
        self.pm = h
        self.device = torch.device("cuda", device)
        self.box = [float(v) for v in box]
        self.G = float(G)

    def accel(self, x, y, z, m, stream=None):
        """Long-range acceleration (3 device tensors) of particles at x, y, z with masses m."""
        n = x.shape[0]
        out = [torch.empty(n, dtype=torch.float32, device=x.device) for _ in range(3)]
        s = stream if stream is not None else torch.cuda.current_stream()
        st = lib().crk_pm_accel(self.pm, C.c_int64(n), *[C.c_void_p(t.data_ptr()) for t in (x, y, z, m, *out)],
                                C.c_void_p(s.cuda_stream))
        if st != 0:
            raise CrkError(st, "crk_pm_accel")
        return out

    def force_profile(self, r, n_dir=16, n_src=4, seed=0):
        """Measured radial force of this mesh per unit source mass and separation,
        f(r) = -a_r / (G r), averaged over ``n_dir`` random directions and ``n_src`` random
        source positions (CIC makes the mesh force depend on the source's sub-cell offset
        and the probe's orientation).  One crk_pm_accel call per source, massless probes.
        HACC fits its short-range polynomial to this measured grid force rather than to the
        analytic one (feed the result to
        ``gen.configs.fit_poly_samples``)."""
        r = np.asarray(r, np.float64)
        rng = np.random.default_rng(seed)
        box = np.asarray(self.box)
        acc = np.zeros(r.shape[0])
        for _ in range(n_src):
            src = rng.random(3) * box
            u = rng.standard_normal((n_dir, 3))
            u /= np.linalg.norm(u, axis=1, keepdims=True)
            d = (r[None, :, None] * u[:, None, :]).reshape(-1, 3)  # (n_dir * len(r), 3)
            pos = np.mod(np.concatenate([src[None], src + d]), box)
            m = np.zeros(pos.shape[0])
            m[0] = 1.0
            t = [torch.tensor(v, dtype=torch.float32, device=self.device)
                 for v in (pos[:, 0], pos[:, 1], pos[:, 2], m)]
            a = torch.stack(self.accel(*t), 1)[1:].double().cpu().numpy()
            # positions are fp32: measure the radial component along the realised separation
            p32 = pos.astype(np.float32).astype(np.float64)
            dd = p32[1:] - p32[0]
            dd -= box * np.round(dd / box)
            rr = np.linalg.norm(dd, axis=1)
            ar = -(a * dd).sum(1) / np.maximum(rr, 1e-30)
            acc += (ar / (self.G * np.maximum(rr, 1e-30))).reshape(n_dir, -1).mean(0)
        return acc / n_src

    def close(self):
        if getattr(self, "pm", None):
            lib().crk_pm_destroy(self.pm)
            self.pm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass



class SlabPM:
    """One rank's share of the slab-decomposed particle mesh (crk_pm_slab_*; include/crksr.h).
    Each method is one C-ABI call on a caller-owned buffer; the collectives between them are
    the caller's (``pm_dist.pm_accel_distributed`` with torch.distributed)."""

    def __init__(self, n_grid: int, box, r_s: float, G: float, rank: int, nranks: int, device=0):
        b = (C.c_double * 3)(*[float(v) for v in box])
        h = C.c_void_p()
        st = lib().crk_pm_slab_create(int(n_grid), b, C.c_float(r_s), C.c_float(G), int(rank), int(nranks),
                                      int(device), C.byref(h))
        if st != 0:
            raise CrkError(st, "crk_pm_slab_create")
        self.pm = h
        self.device = torch.device("cuda", device)
        self.n, self.rank, self.P = int(n_grid), int(rank), int(nranks)
        self.nl = self.n // self.P
        self.nzc = self.n // 2 + 1

    # buffer shapes (include/crksr.h)
    def sizes(self):
        n, nl, P, nzc = self.n, self.nl, self.P, self.nzc
        return dict(rho_full=n ** 3, rho_slab=nl * n * n, send=P * nl * nl * nzc, send3=P * 3 * nl * nl * nzc,
                    acc_slab=3 * nl * n * n)

    @staticmethod
    def _s(stream):
        return C.c_void_p((stream if stream is not None else torch.cuda.current_stream()).cuda_stream)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    def _ck(self, st, what):
        if st != 0:
            raise CrkError(st, what)

    def deposit(self, x, y, z, m, stream=None):
        rho = torch.empty(self.sizes()["rho_full"], dtype=torch.float32, device=self.device)
        self._ck(lib().crk_pm_deposit(self.pm, C.c_int64(x.shape[0]), *map(self._p, (x, y, z, m, rho)),
                                      self._s(stream)), "crk_pm_deposit")
        return rho

    def forward(self, rho_slab, stream=None):
        send = torch.empty(self.sizes()["send"], dtype=torch.complex64, device=self.device)
        self._ck(lib().crk_pm_slab_forward(self.pm, self._p(rho_slab), self._p(send), self._s(stream)),
                 "crk_pm_slab_forward")
        return send

    def solve(self, recv, stream=None):
        send3 = torch.empty(self.sizes()["send3"], dtype=torch.complex64, device=self.device)
        self._ck(lib().crk_pm_slab_solve(self.pm, self._p(recv), self._p(send3), self._s(stream)),
                 "crk_pm_slab_solve")
        return send3

    def inverse(self, recv3, stream=None):
        acc = torch.empty(self.sizes()["acc_slab"], dtype=torch.float32, device=self.device)
        self._ck(lib().crk_pm_slab_inverse(self.pm, self._p(recv3), self._p(acc), self._s(stream)),
                 "crk_pm_slab_inverse")
        return acc

    def interp(self, x, y, z, acc_full, stream=None):
        out = [torch.empty(x.shape[0], dtype=torch.float32, device=self.device) for _ in range(3)]
        self._ck(lib().crk_pm_interp(self.pm, C.c_int64(x.shape[0]), *map(self._p, (x, y, z, acc_full, *out)),
                                     self._s(stream)), "crk_pm_interp")
        return out

    def close(self):
        if getattr(self, "pm", None):
            lib().crk_pm_destroy(self.pm)
            self.pm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
