"""Slab-decomposed long-range particle mesh over ranks (cuFFT with
NCCL all-to-all; include/crksr.h "slab-decomposed particle mesh").

The kernels are the crk_pm_slab_* calls (``SlabPM``); this module only sequences them with
the four collectives between them — a reduce-scatter of the deposited mesh, two all-to-all
transposes and an all-gather of the acceleration slabs — through a ``comm`` object, so the
same sequence runs over torch.distributed (NCCL) or, in the tests, over P ranks emulated
on one GPU.
"""
from __future__ import annotations

import contextlib

import torch


class TorchComm:
    """The four collectives over torch.distributed (NCCL on B200)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group

    def reduce_scatter(self, out, full):
        self.dist.reduce_scatter_tensor(out, full, group=self.group)

    def all_to_all(self, out, inp):
        self.dist.all_to_all_single(out, inp, group=self.group)

    def all_gather(self, out, part):
        self.dist.all_gather_into_tensor(out, part, group=self.group)


class HostStagedComm(TorchComm):
    """The same collectives over a CPU backend (gloo): device tensors are staged through host
    memory.  For checking the distributed sequence with several processes on one GPU."""

    def _run(self, fn, out, *inp):
        o = out.cpu()
        fn(o, *[t.cpu() for t in inp], group=self.group)
        out.copy_(o)

    def reduce_scatter(self, out, full):
        # gloo has no reduce-scatter of complex/large tensors on every build: all-reduce + chunk
        f = full.to("cpu", copy=True)
        self.dist.all_reduce(f, group=self.group)
        out.copy_(f.chunk(self.dist.get_world_size(self.group))[self.dist.get_rank(self.group)])

    def all_to_all(self, out, inp):
        self._run(self.dist.all_to_all_single, out, inp)

    def all_gather(self, out, part):
        self._run(self.dist.all_gather_into_tensor, out, part)


# ---- the collectives' semantics on P emulated ranks (lists indexed by rank) ----
def emu_reduce_scatter(full):
    P = len(full)
    return [c.contiguous() for c in torch.stack(full).sum(0).chunk(P)]


def emu_all_to_all(inp):
    P = len(inp)
    return [torch.cat([inp[q].chunk(P)[r] for q in range(P)]) for r in range(P)]


def emu_all_gather(parts):
    return torch.cat(parts)


def pm_accel_distributed(spm, x, y, z, m, comm=None, stream=None):
    """Long-range acceleration of this rank's particles (x, y, z, m device tensors) with the
    mesh slab-decomposed over the ranks of ``comm`` (default: the torch.distributed world).

    Everything — the SlabPM kernels, the collectives and the buffers' allocations — is
    issued on ONE stream, ``stream`` (default: the current stream), made current for the
    whole sequence: torch.distributed orders its collectives after the current stream's
    work, and the caching allocator ties each buffer to the stream that allocated it, so no
    kernel can read a buffer before the collective that fills it lands, nor a buffer be
    reused while a collective still reads it.  The caller's inputs must be ready on
    ``stream`` (it waits for the current stream when a different one is given)."""
    comm = comm or TorchComm()
    sz = spm.sizes()
    on_gpu = x.device.type == "cuda"  # (CPU tensors: the test doubles of tests/test_pm.py)
    if on_gpu and stream is not None:
        stream.wait_stream(torch.cuda.current_stream(x.device))
    with torch.cuda.stream(stream) if on_gpu and stream is not None else contextlib.nullcontext():
        rho = spm.deposit(x, y, z, m)
        rho_slab = torch.empty(sz["rho_slab"], dtype=torch.float32, device=rho.device)
        comm.reduce_scatter(rho_slab, rho)
        send = spm.forward(rho_slab)
        recv = torch.empty_like(send)
        comm.all_to_all(recv, send)
        send3 = spm.solve(recv)
        recv3 = torch.empty_like(send3)
        comm.all_to_all(recv3, send3)
        acc = spm.inverse(recv3)
        acc_full = torch.empty(spm.P * acc.numel(), dtype=torch.float32, device=acc.device)
        comm.all_gather(acc_full, acc)
        out = spm.interp(x, y, z, acc_full)
    if on_gpu and stream is not None:
        for t in (x, y, z, *out):
            t.record_stream(stream)
    return out


def pm_accel_emulated(spms, parts):
    """P ranks emulated on one device, phase by phase (the collectives as tensor copies):
    ``spms[r]`` is rank r's SlabPM, ``parts[r]`` its (x, y, z, m).  Returns each rank's
    accelerations; for tests and single-GPU checks of the decomposed path."""
    slabs = emu_reduce_scatter([s.deposit(*p) for s, p in zip(spms, parts)])
    recv = emu_all_to_all([s.forward(slabs[r]) for r, s in enumerate(spms)])
    recv3 = emu_all_to_all([s.solve(recv[r]) for r, s in enumerate(spms)])
    acc_full = emu_all_gather([s.inverse(recv3[r]) for r, s in enumerate(spms)])
    return [s.interp(p[0], p[1], p[2], acc_full) for s, p in zip(spms, parts)]
