"""3-D domain decomposition with leaf-granular ghost exchange.

Host-side plumbing only: the decomposition and the cell masks are small host logic;
the selection, packing and unpacking run in libcrksr.so (crk_select_cells /
crk_select_gas / crk_pack_* / crk_unpack_*) and the transfers are NCCL send/recv
through torch.distributed (batch_isend_irecv).  The paper runs one MPI rank per GPU
 but does not describe the exchange; this follows north_star's
"3-D spatial domain decomposition with overload/ghost zones refreshed by send/recv".

Per substep (rank r owning the chaining-mesh cells D_r):
  R1  own particles in D_r ∩ halo_h(D_s) -> peer s (48-byte records); build lists over
      own + ghosts with i-leaves only in D_r (so lists = the global lists' own rows);
  gravity (i-centric), geometry;
  R2  V of own gas in D_r ∩ halo_h(D_s) -> peer s (order: gas rank = key order on both);
  corrections, extras;
  R3  accel records of the same gas -> peer s;
  accel / du-dt.
halo width h = ceil(reach / cell_side), reach = max(r_c, H_max) (1 + 2^-20) with H_max the
global maximum smoothing length (one all-reduce).
"""
from __future__ import annotations

import math

import numpy as np
import torch

from .binding import Particles, Solver

GRIDS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}


def grid_dims(P: int):
    if P in GRIDS:
        return GRIDS[P]
    raise ValueError("ranks must be 1, 2, 4 or 8 (2x1x1, 2x2x1, 2x2x2 decompositions)")


class Decomposition:
    """Split the periodic box's chaining-mesh cells into P equal bricks."""

    def __init__(self, params: dict, P: int):
        self.params = params
        self.P = P
        self.dims = grid_dims(P)
        cs = params["cell_side"]
        self.ncell = [int(round(b / cs)) for b in params["box"]]
        for a in range(3):
            if self.ncell[a] % self.dims[a]:
                raise ValueError("cells per axis must divide evenly among the ranks")
        self.lo, self.hi = [], []
        for r in range(P):
            c = (r % self.dims[0], (r // self.dims[0]) % self.dims[1], r // (self.dims[0] * self.dims[1]))
            w = [self.ncell[a] // self.dims[a] for a in range(3)]
            self.lo.append([c[a] * w[a] for a in range(3)])
            self.hi.append([(c[a] + 1) * w[a] for a in range(3)])

    def rank_params(self, r: int) -> dict:
        p = dict(self.params)
        if self.P > 1:
            p["dom_lo"], p["dom_hi"] = list(self.lo[r]), list(self.hi[r])
        return p

    def halo_width(self, hmax2: float) -> int:
        reach = math.sqrt(max(self.params["rcut2"], hmax2)) * (1.0 + 2.0**-20) * (1.0 + 1e-9)
        return int(math.ceil(reach / self.params["cell_side"]))

    def owner_of_cells(self, cx, cy, cz):
        w = [self.ncell[a] // self.dims[a] for a in range(3)]
        return (cx // w[0]) + self.dims[0] * ((cy // w[1]) + self.dims[1] * (cz // w[2]))

    def masks(self, recv: int, send: int, h: int):
        """Per-axis cell masks of D_send ∩ halo_h(D_recv) (periodic); None when empty."""
        out = []
        for a in range(3):
            n = self.ncell[a]
            m = np.zeros(n, np.uint8)
            lo, hi = self.lo[recv][a], self.hi[recv][a]
            for c in range(lo - h, hi + h):
                m[c % n] = 1
            own = np.zeros(n, np.uint8)
            own[self.lo[send][a]:self.hi[send][a]] = 1
            m &= own
            if not m.any():
                return None
            out.append(m)
        return out

    def cells_of(self, parts: dict):
        q = max(self.params["box"]) * 2.0**-23
        cs = int(round(math.log2(self.params["cell_side"] / q)))
        return [(np.asarray(parts[k], np.float64) / q).astype(np.int64) >> cs for k in "xyz"]

    def split(self, parts: dict, r: int) -> dict:
        """The particles of a global (host) set that rank r owns."""
        cx, cy, cz = self.cells_of(parts)
        keep = self.owner_of_cells(cx, cy, cz) == r
        return {k: np.ascontiguousarray(v[keep]) for k, v in parts.items()}


# ---------------------------------------------------------------- exchanges
class DistExchange:
    """Peer-to-peer exchange over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, rank: int, world: int, device):
        self.rank, self.world, self.device = rank, world, torch.device(device)

    def _p2p(self, sends: dict, recvs: dict):
        import torch.distributed as dist

        host = dist.get_backend() == "gloo" and self.device.type == "cuda"  # gloo moves host tensors
        if host:
            sends = {s: t.cpu() for s, t in sends.items()}
            dev_recvs, recvs = recvs, {s: torch.empty(t.shape, dtype=t.dtype) for s, t in recvs.items()}
        ops = []
        for s, t in sends.items():
            ops.append(dist.P2POp(dist.isend, t, s))
        for s, t in recvs.items():
            ops.append(dist.P2POp(dist.irecv, t, s))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if host:
            for s, t in recvs.items():
                dev_recvs[s].copy_(t)

    def alltoallv(self, sends: dict, width: int, dtype=torch.float32) -> dict:
        """sends: {peer: tensor (n, width)} -> {peer: tensor (m, width)} (counts exchanged first)."""
        peers = [s for s in range(self.world) if s != self.rank]
        cnt_out = {s: torch.tensor([sends[s].shape[0] if s in sends else 0], dtype=torch.int64,
                                   device=self.device) for s in peers}
        cnt_in = {s: torch.zeros(1, dtype=torch.int64, device=self.device) for s in peers}
        self._p2p(cnt_out, cnt_in)
        outs = {s: sends[s].contiguous() for s in peers if s in sends and sends[s].shape[0] > 0}
        ins = {s: torch.empty((int(cnt_in[s].item()), width), dtype=dtype, device=self.device)
               for s in peers if int(cnt_in[s].item()) > 0}
        self._p2p(outs, ins)
        return ins

    def allreduce_max(self, v: float) -> float:
        import torch.distributed as dist

        dev = "cpu" if dist.get_backend() == "gloo" else self.device
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())


class DomainRank:
    """One rank's share of a decomposed substep, in phases (so that ranks can also be
    emulated in one process on one device)."""

    def __init__(self, decomp: Decomposition, r: int, own: dict, device, stream=None, outputs=True):
        self.outputs = outputs  # Particles outputs of the local set ("forces": results only)
        self.d, self.r, self.device = decomp, r, torch.device(device)
        self.params = decomp.rank_params(r)
        self.own_host = own
        self.n_own = own["x"].shape[0]
        self.own = Particles.from_host(own, self.device, outputs=False)
        self.solver = Solver(self.params, self.device.index if self.device.index is not None else 0)
        self.stream = stream
        self.h = None

    def local_hmax2(self) -> float:
        gas = self.own_host["species"] == 1
        if not gas.any():
            return 0.0
        return float((self.own_host["H"][gas].astype(np.float32) ** 2).max())

    # R1 ---------------------------------------------------------------
    def r1_pack(self, h: int) -> dict:
        self.h = h
        out = {}
        for s in range(self.d.P):
            if s == self.r:
                continue
            m = self.d.masks(recv=s, send=self.r, h=h)
            if m is None:
                continue
            idx = self.solver.select_cells(self.own, m, n=self.n_own, stream=self.stream)
            out[s] = self.solver.pack_particles(self.own, idx, stream=self.stream)
        return out

    def r1_unpack_and_build(self, recv: dict):
        n_ghost = sum(int(t.shape[0]) for t in recv.values())
        self.n_total = self.n_own + n_ghost
        p = Particles(self.n_total, self.device, self.outputs)
        for k in Particles.IN_F32 + ("species", "id"):
            getattr(p, k)[: self.n_own].copy_(getattr(self.own, k))
        off = self.n_own
        for s in sorted(recv):
            self.solver.unpack_particles(p, off, recv[s], stream=self.stream)
            off += recv[s].shape[0]
        self.p = p
        self._gl = None
        self.solver.build_lists(p, self.stream)

    # passes -------------------------------------------------------------
    def gravity_geometry(self, dt_grav=0.0):
        self.solver.gravity_kick(self.p, dt_grav, self.stream)
        self.solver.geometry(self.p, self.stream)

    def _gas_lists(self):
        if getattr(self, "_gl", None) is None:
            self._gl = {}
            ng = self.n_total  # capacity bound
            for s in range(self.d.P):
                if s == self.r:
                    continue
                ms = self.d.masks(recv=s, send=self.r, h=self.h)
                mr = self.d.masks(recv=self.r, send=s, h=self.h)
                send = self.solver.select_gas(ms, self.device, self.stream, ng) if ms is not None else None
                rec = self.solver.select_gas(mr, self.device, self.stream, ng) if mr is not None else None
                self._gl[s] = (send, rec)
        return self._gl

    def r2_pack(self) -> dict:
        return {s: self.solver.pack_gas(0, send, self.stream) for s, (send, _) in self._gas_lists().items()
                if send is not None and send.numel() > 0}

    def r2_unpack(self, recv: dict):
        for s, buf in recv.items():
            idx = self._gas_lists()[s][1]
            assert idx is not None and idx.numel() == buf.shape[0], "R2 message does not match the ghost set"
            self.solver.unpack_gas(0, idx, buf, self.stream)

    def corrections_extras(self):
        self.solver.corrections_extras(self.p, self.stream)

    def r3_pack(self) -> dict:
        return {s: self.solver.pack_gas(1, send, self.stream) for s, (send, _) in self._gas_lists().items()
                if send is not None and send.numel() > 0}

    def r3_unpack(self, recv: dict):
        for s, buf in recv.items():
            idx = self._gas_lists()[s][1]
            assert idx is not None and idx.numel() == buf.shape[0], "R3 message does not match the ghost set"
            self.solver.unpack_gas(1, idx, buf, self.stream)

    def accel(self, dt_hydro=0.0):
        self.solver.hydro_accel_dudt(self.p, dt_hydro, self.stream)

    def own_mask(self) -> torch.Tensor:
        """Sorted positions holding own particles (inputs 0..n_own-1 are own)."""
        return self.p.perm < self.n_own

    def close(self):
        self.solver.close()


def substep_inprocess(ranks, dt_grav=0.0, dt_hydro=0.0):
    """Run one decomposed substep for ranks emulated sequentially in one process (tests)."""
    hmax2 = max(rk.local_hmax2() for rk in ranks)
    h = ranks[0].d.halo_width(hmax2)
    sends = [rk.r1_pack(h) for rk in ranks]
    for rk in ranks:
        rk.r1_unpack_and_build({s: sends[s][rk.r] for s in range(len(ranks)) if rk.r in sends[s]})
    for rk in ranks:
        rk.gravity_geometry(dt_grav)
    sends = [rk.r2_pack() for rk in ranks]
    for rk in ranks:
        rk.r2_unpack({s: sends[s][rk.r] for s in range(len(ranks)) if rk.r in sends[s]})
    for rk in ranks:
        rk.corrections_extras()
    sends = [rk.r3_pack() for rk in ranks]
    for rk in ranks:
        rk.r3_unpack({s: sends[s][rk.r] for s in range(len(ranks)) if rk.r in sends[s]})
    for rk in ranks:
        rk.accel(dt_hydro)


def substep_dist(rk: DomainRank, ex: DistExchange, dt_grav=0.0, dt_hydro=0.0, hmax2=None):
    """One decomposed substep on this rank, exchanging with the other ranks."""
    if hmax2 is None:
        hmax2 = ex.allreduce_max(rk.local_hmax2())
    h = rk.d.halo_width(hmax2)
    rk.r1_unpack_and_build(ex.alltoallv(rk.r1_pack(h), 12))
    rk.gravity_geometry(dt_grav)
    rk.r2_unpack(ex.alltoallv(rk.r2_pack(), 1))
    rk.corrections_extras()
    rk.r3_unpack(ex.alltoallv(rk.r3_pack(), 36))
    rk.accel(dt_hydro)
