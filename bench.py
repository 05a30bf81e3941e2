#!/usr/bin/env python
"""Benchmark of the CRK-HACC short-range substep on B200 (BASELINE.json metric:
pair interactions/s and short-range substep time; % of FP32 peak).

A step = one whole short-range substep: build lists (sort,
leaves, lists), gravity + kick, geometry, corrections, extras, accel/du-dt, over the
device-resident 2x256^3 perturbed-lattice workload (config 4 at 1 GPU = config 5's
per-GPU size).  Prints ONE JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# canonical flop per ordered pair (FMA = 2, MUFU = 1, compare/select = 0)
FLOP_PER_PAIR = {"gravity": 30, "geometry": 22, "corrections_extras": 114 + 103, "accel_dudt": 256}
PASSES = ["build_lists", "gravity", "geometry", "corrections_extras", "accel_dudt"]
# the kernel that dominates each pass (profiles/r01/ncu_traffic.json is matched against it)
_DOM_KERNEL = {"gravity": "grav_pipe_kernel", "geometry": "pair_kernel<GeoPass", "corrections_extras": "list_kernel2<",
               "accel_dudt": "list_kernel<AccPass"}
METRIC = "pair interactions/s & short-range substep time at 1/2/4/8 B200; % FP32 peak"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a moment to start: wait for its first sample, then keep only
            # the samples taken from here on (the timed region)
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.02)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_sample(parts, params, n_grav=20000, n_gas=1500, seed=1):
    """Time the fp64 oracle as it stands on a bounded sample of the workload; returns
    (pair interactions evaluated, seconds, description, mean pair interactions per particle).
    The pairs are counted by the oracle itself (oracle.counts on the sampled sets, outside the
    timed region): no GPU library is involved."""
    import oracle

    rng = np.random.default_rng(seed)
    n = parts["x"].shape[0]
    gas = np.nonzero(parts["species"] == 1)[0]
    tg = np.sort(rng.choice(gas, min(n_gas, gas.shape[0]), replace=False))
    ta = np.sort(rng.choice(n, min(n_grav, n), replace=False))
    t0 = time.perf_counter()
    oracle.gravity(parts, params, ta)
    off, nb = oracle.neighbour_sets(parts, params, tg, 2)
    T2 = np.unique(np.concatenate([tg, nb]))
    off, nb = oracle.neighbour_sets(parts, params, T2, 1)
    T1 = np.unique(np.concatenate([T2, nb]))
    V = np.full(n, np.nan)
    V[T1] = oracle.geometry(parts, params, T1)
    cr = oracle.corrections(parts, params, V, T2)
    A, B, dA, dB = np.full(n, np.nan), np.full((n, 3), np.nan), np.full((n, 3), np.nan), np.full((n, 9), np.nan)
    A[T2], B[T2], dA[T2], dB[T2] = cr["A"], cr["B"], cr["dA"], cr["dB"]
    ex = oracle.extras(parts, params, V, A, B, dA, dB, T2)
    rho, P, c, dv = np.full(n, np.nan), np.full(n, np.nan), np.full(n, np.nan), np.full((n, 9), np.nan)
    rho[T2], P[T2], c[T2], dv[T2] = ex["rho"], ex["P"], ex["cs"], ex["dv"]
    oracle.accel(parts, params, V, A, B, dA, dB, rho, P, c, dv, tg)
    secs = time.perf_counter() - t0
    c_a = oracle.counts(parts, params, ta)
    c_1 = oracle.counts(parts, params, T1)
    c_2 = oracle.counts(parts, params, T2)
    c_g = oracle.counts(parts, params, tg)
    pairs = (int(c_a["grav"].sum()) + int(c_1["gather"].sum()) + 2 * int(c_2["gather"].sum())
             + int(c_g["sym"].sum()))
    # per-particle means of the sampled sets -> the whole workload's pair interactions
    gas_frac = gas.shape[0] / n
    per_particle = (c_a["grav"].mean() + gas_frac * (3 * c_g["gather"].mean() + c_g["sym"].mean()))
    desc = (f"oracle (fp64 C, OpenMP) on {ta.shape[0]} gravity targets + hydro chain for {tg.shape[0]} gas "
            f"targets (closure {T1.shape[0]}/{T2.shape[0]}); pairs counted by oracle.counts on the computed sets")
    return pairs, secs, desc, float(per_particle)


def oracle_1core_c1():
    """the config-1 oracle ("CPU oracle in seconds") on ONE core — the
    whole substep (gravity, geometry, corrections, extras, accel/du-dt) plus the counts."""
    import oracle
    from gen import make_config

    p1, q1 = make_config("c1")
    n0 = oracle.num_threads()
    oracle.set_threads(1)
    try:
        t0 = time.perf_counter()
        oracle.substep(p1, q1)
        oracle.counts(p1, q1)
        return time.perf_counter() - t0
    finally:
        oracle.set_threads(n0)


def run_reference(args, parts, params, rank, world):
    """--impl reference: the oracle (fp64 CPU) timed on this host's cores, rank 0 only.  No
    GPU library is loaded on this path: pairs are counted by the oracle."""
    import oracle

    if rank != 0:
        return
    times, pairs_tot, pp = [], 0, []
    for s in range(args.warmup + args.steps):
        pairs, secs, desc, per_particle = oracle_sample(parts, params, n_grav=4000, n_gas=300, seed=100 + s)
        if s >= args.warmup:
            times.append(secs)
            pairs_tot += pairs
            pp.append(per_particle)
    val = pairs_tot / sum(times)
    n = parts["x"].shape[0]
    # one whole substep of this workload at the oracle's measured rate (pair interactions per
    # substep estimated from the sampled per-particle counts)
    ms = 1e3 * float(np.mean(pp)) * n / val
    line = {"metric": METRIC, "impl": "reference", "value": val, "unit": "pair interactions/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "ms_per_step_basis": "one whole substep of the workload at the measured rate (pairs per substep "
                                 "from the sampled per-particle oracle counts); each timed step is a bounded sample",
            "sample_ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config(args, parts),
            "cpu_baseline": {"value": val, "unit": "pair interactions/s", "cores": oracle.num_threads(),
                             "kind": "oracle", "sample": desc, "cpu": _cpu_model()},
            "e2e": {"value": val, "unit": "pair interactions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(args, parts):
    n = parts["x"].shape[0]
    return {"workload": f"{args.config}: 2x{round((n / 2) ** (1 / 3))}^3 DM+gas perturbed lattice (Zel'dovich rms 0.1), "
                        "periodic box, one gravity + CRK-SPH short-range substep",
            "particles_per_gpu": n, "l2": "inputs (>1.5 GB) larger than L2", "seq_len": None,
            "outputs": "a_grav, a_hydro, du/dt per particle (CRK intermediates computed, not copied out)",
            "streams": "gravity (a3) || geometry (a4) on two streams" if getattr(args, "overlap", False) else "one",
            "order": "SoA sorted in place: timed steps see the previous step's order (e2e: random order each step)"}


_COUNT_CACHE = {}


def _counts_input_order(parts, params):
    import torch
    from paper_2310_16122_b200 import Particles, Solver

    key = id(parts)
    if key in _COUNT_CACHE:
        return _COUNT_CACHE[key]
    p = Particles.from_host(parts, "cuda", outputs=False)
    s = Solver(params, torch.cuda.current_device())
    s.build_lists(p)
    s.geometry(p)  # builds the neighbour lists: the gas counts come from the list walks the passes make
    cg, ch, cs = s.count_pairs(p)
    perm = p.perm.cpu().numpy().astype(np.int64)
    out = []
    for c in (cg, ch, cs):
        o = np.empty(p.n, np.int64)
        o[perm] = c.cpu().numpy()
        out.append(o)
    s.close()
    del p
    torch.cuda.empty_cache()
    _COUNT_CACHE[key] = tuple(out)
    return _COUNT_CACHE[key]


def tile_config(parts, params, P, r):
    """Weak scaling: the single-GPU workload tiled over the 2x1x1 / 2x2x1 / 2x2x2 rank grid
    (periodic replicas, so the generator's H stays exact); rank r gets tile r on the global
    box's quantum q = L_max 2^-23 (the tile is put on that quantum first, so the tiles are exact
    shifted copies), ids offset by r n."""
    from gen.configs import make_params, quantise
    from paper_2310_16122_b200.domain import grid_dims

    dims = grid_dims(P)
    box = [params["box"][a] * dims[a] for a in range(3)]
    gp = make_params(box, poly=params["poly"], symmetric=params.get("symmetric", 1))
    c = (r % dims[0], (r // dims[0]) % dims[1], r // (dims[0] * dims[1]))
    # the tile on the global box's quantum first (wrapped into the tile), so every rank's tile
    # is an exact shifted copy: the global system is a periodic replica bit for bit
    base = np.stack([parts[k].astype(np.float64) for k in "xyz"], 1)
    base = quantise(quantise(base, box).astype(np.float64), params["box"]).astype(np.float64)
    pos = quantise(base + np.asarray(c, np.float64) * np.asarray(params["box"]), box)
    own = dict(parts)
    own["x"], own["y"], own["z"] = (np.ascontiguousarray(pos[:, a]) for a in range(3))
    own["id"] = parts["id"] + r * parts["x"].shape[0]
    return own, gp


def _e2e_multi(args, rk, ex, own, dev, hmax2, overlap, red_dev):
    """e2e at N > 1 through the public API: every step, each rank copies its own particles' inputs
    up from pinned host memory (into the second of two own sets, during the previous step) and its
    local set's results down (snapshotted on the device at the end of the step, then copied on a
    second copy stream during the next one).  Returns (max-over-ranks ms per step, (h2d, d2h)
    bytes per step of this rank) or (None, None) if it fails."""
    import torch
    import torch.distributed as dist
    from paper_2310_16122_b200 import Particles
    from paper_2310_16122_b200.domain import substep_dist

    try:
        host = {k: torch.from_numpy(np.ascontiguousarray(own[k])).pin_memory()
                for k in Particles.IN_F32 + ("species", "id")}
        bi = sum(t.numel() * t.element_size() for t in host.values())
        outk = list(Particles.FORCES) + ["perm"]
        # two own sets of our own (rk.own may be a view into the rank's carried local set)
        owns = [Particles(rk.n_own, dev, outputs=False), Particles(rk.n_own, dev, outputs=False)]
        stream = torch.cuda.current_stream(dev)
        h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_done = [torch.cuda.Event(), torch.cuda.Event()]
        ev_out = [torch.cuda.Event(), torch.cuda.Event()]
        snap, hout = [None, None], [None, None]
        nbytes = [0]

        def run(nsteps):
            h2d.wait_stream(stream)
            with torch.cuda.stream(h2d):
                owns[0].load(host, non_blocking=True)
            ev_in[0].record(h2d)
            for k in range(nsteps):
                b = k % 2
                stream.wait_event(ev_in[b])
                rk.own = owns[b]
                substep_dist(rk, ex, 0.0, 0.0, hmax2, overlap=overlap)
                n = rk.n_total
                if snap[b] is None or snap[b][0].shape[0] < n:
                    snap[b] = [torch.empty(int(1.1 * n) + 16, dtype=getattr(rk.p, key).dtype, device=dev)
                               for key in outk]
                    hout[b] = [torch.empty(t.shape[0], dtype=t.dtype).pin_memory() for t in snap[b]]
                if k >= 2:
                    stream.wait_event(ev_out[b])  # step k-2's results of this snapshot are down
                for t, key in zip(snap[b], outk):
                    t[:n].copy_(getattr(rk.p, key)[:n])
                ev_done[b].record(stream)
                if k + 1 < nsteps:
                    nb = (k + 1) % 2
                    if k >= 1:
                        h2d.wait_event(ev_done[nb])  # step k - 1 is done with that set's inputs
                    with torch.cuda.stream(h2d):
                        owns[nb].load(host, non_blocking=True)
                    ev_in[nb].record(h2d)
                d2h.wait_event(ev_done[b])
                with torch.cuda.stream(d2h):
                    for t, h in zip(snap[b], hout[b]):
                        h[:n].copy_(t[:n], non_blocking=True)
                ev_out[b].record(d2h)
                nbytes[0] = sum(n * t.element_size() for t in snap[b])
            stream.wait_stream(d2h)

        run(2)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=red_dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        rk.own = owns[0]
        return float(ms.item()), (bi, nbytes[0])
    except Exception as exc:  # pragma: no cover
        print(f"e2e (N > 1) failed: {exc}", file=sys.stderr)
        return None, None


def run_multi(args, parts, params, rank, world, local, gen_s):
    """N > 1: 3-D domain decomposition, ghost exchange over NCCL, weak scaling."""
    import torch
    import torch.distributed as dist
    from paper_2310_16122_b200.domain import Decomposition, DistExchange, DomainRank, substep_dist

    own, gp = tile_config(parts, params, world, rank)
    d = Decomposition(gp, world)
    dev = torch.device("cuda", local)
    rk = DomainRank(d, rank, own, dev, outputs="forces")
    ex = DistExchange(rank, world, dev)
    hmax2 = ex.allreduce_max(rk.local_hmax2())
    # overlapped R2/R3 exchange: on with NCCL by default; CRK_OVERLAP=1/0 forces it (tests: gloo ranks)
    overlap = {"1": True, "0": False}.get(os.environ.get("CRK_OVERLAP", ""))
    for _ in range(args.warmup):
        substep_dist(rk, ex, args.dt, args.dt, hmax2, overlap=overlap)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = rk.solver.launch_count()
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            substep_dist(rk, ex, args.dt, args.dt, hmax2, overlap=overlap)
        e1.record()
        torch.cuda.synchronize()
    red_dev = "cpu" if dist.get_backend() == "gloo" else dev
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=red_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    launches = (rk.solver.launch_count() - l0) // max(args.steps, 1)
    e2e_ms, e2e_bytes = _e2e_multi(args, rk, ex, own, dev, hmax2, overlap, red_dev)
    cg, ch, cs = rk.solver.count_pairs(rk.p)
    own_m = rk.own_mask()
    pr = torch.tensor([int(cg[own_m].sum()), int(ch[own_m].sum()), int(cs[own_m].sum()),
                       int(rk.n_total - rk.n_own)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(pr)
    pair_int = pr[0].item() + 3 * pr[1].item() + pr[2].item()
    ms_step = float(ms.item())
    if rank == 0:
        line = {"metric": METRIC, "value": pair_int / (ms_step * 1e-3), "unit": "pair interactions/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": dict(_config(args, parts), parallelism=f"3-D domain decomposition {d.dims}, "
                               f"ghost exchange R1/R2/R3 over {dist.get_backend()} send/recv"
                               + (", R2/R3 overlapped with the interior rows" if (overlap if overlap is not None else
                                                                                  dist.get_backend() == "nccl") else ""),
                               global_box=gp["box"],
                               ghost_particles_total=int(pr[3].item()), generator_s=round(gen_s, 1)),
                "substep_ms": ms_step,
                "pairs": {"gravity": int(pr[0].item()), "gather": int(pr[1].item()), "sym": int(pr[2].item())},
                "pair_interactions_per_step": int(pair_int),
                "clocks": clk.summary(), "gpu_launches": int(launches),
                "e2e": None if e2e_ms is None else {
                    "value": pair_int / (e2e_ms * 1e-3), "unit": "pair interactions/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": e2e_bytes[0], "d2h_bytes_per_step": e2e_bytes[1],
                    "bytes_basis": "rank 0's own-particle inputs up, its local set's results down (every rank does "
                                   "the same on its own link); time = max over ranks",
                    "overlap": "per rank: H2D of step k+1 into a second own set and D2H of step k's results "
                               "(snapshotted on the device) on two copy streams during the next step"},
                "cpu_baseline": None, "roofline": None}
        print(json.dumps(line), flush=True)
    rk.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dt", type=float, default=0.0)
    ap.add_argument("--overlap", action="store_true",
                    help="gravity on a side stream concurrently with geometry (measured: no gain, 53.6 ms either way)")
    ap.add_argument("--symmetric", type=int, default=None,
                    help="kernel variant bitmask: 1 = Newton-3 gravity, 2 = Newton-3 accel (default: library default)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("CRK_DIST_BACKEND", "nccl")  # gloo: ranks sharing one GPU (tests)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if os.environ.get("CRK_SHARE_GPU"):
        local = 0
    torch.cuda.set_device(local)

    from gen import make_config

    t0 = time.perf_counter()
    parts, params = make_config(args.config)
    if args.symmetric is not None:
        params["symmetric"] = args.symmetric
    gen_s = time.perf_counter() - t0

    if args.impl == "reference":
        run_reference(args, parts, params, rank, world)
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    if world > 1:
        run_multi(args, parts, params, rank, world, local, gen_s)
        import torch.distributed as dist

        dist.destroy_process_group()
        return

    from paper_2310_16122_b200 import Particles, Solver

    dev = torch.device("cuda", local)
    # a created (non-legacy-default) stream: the legacy default stream would serialise with
    # the e2e copy streams
    stream = torch.cuda.Stream(dev)
    cnts = _counts_input_order(parts, params)
    pairs = {"gravity": int(cnts[0].sum()), "gather": int(cnts[1].sum()), "sym": int(cnts[2].sum())}
    pair_int = pairs["gravity"] + 3 * pairs["gather"] + pairs["sym"]

    # the substep's results (gravity + hydro accelerations, du/dt); the CRK intermediates stay in
    # the library's scratch (the parity tests request and check them)
    p = Particles.from_host(parts, dev, outputs="forces")
    torch.cuda.synchronize()
    solver = Solver(params, local)
    ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in PASSES}
    side = torch.cuda.Stream(dev) if args.overlap else None

    def step(timed, pp=None, grav_done=None):
        p_ = p if pp is None else pp
        if timed:
            ev["build_lists"][0].record(stream)
        solver.build_lists(p_, stream)
        if timed:
            ev["build_lists"][1].record(stream)
        # a3 (gravity) and a4 (geometry) are independent: gravity on a side stream, joined
        # before a5/a6, which read the kicked v (crksr.h); only with --overlap
        gs = side if side is not None else stream
        if side is not None:
            side.wait_stream(stream)
        if timed:
            ev["gravity"][0].record(gs)
        solver.gravity_kick(p_, args.dt, gs)
        if grav_done is not None:  # e2e: the gravity results (and perm) can go down from here on
            grav_done.record(gs)
        if timed:
            ev["gravity"][1].record(gs)
            ev["geometry"][0].record(stream)
        solver.geometry(p_, stream)
        if timed:
            ev["geometry"][1].record(stream)
        if side is not None:
            stream.wait_stream(side)
        if timed:
            ev["corrections_extras"][0].record(stream)
        solver.corrections_extras(p_, stream)  # a5 + a6 fused (crk_corrections_extras)
        if timed:
            ev["corrections_extras"][1].record(stream)
            ev["accel_dudt"][0].record(stream)
        solver.hydro_accel_dudt(p_, args.dt, stream)
        if timed:
            ev["accel_dudt"][1].record(stream)

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    pass_ms = {k: 0.0 for k in PASSES}
    l0 = solver.launch_count()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t_start.record(stream)
        for _ in range(args.steps):
            step(True)
            torch.cuda.synchronize()
            for k in PASSES:
                pass_ms[k] += ev[k][0].elapsed_time(ev[k][1])
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = (solver.launch_count() - l0) // max(args.steps, 1)
    total_ms = t_start.elapsed_time(t_end)
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / args.steps
    for k in pass_ms:
        pass_ms[k] /= args.steps
    value = pair_int * world / (ms_step * 1e-3)

    # dominant kernel roofline (FP32 ALU)
    pk = _peaks()
    props = torch.cuda.get_device_properties(dev)
    n_sm = props.multi_processor_count
    f_max = float(pk.get("sm_max_mhz", 1965.0))
    peak_tf = n_sm * 128 * 2 * f_max * 1e6 / 1e12
    pass_pairs = {"gravity": pairs["gravity"], "geometry": pairs["gather"], "corrections_extras": pairs["gather"],
                  "accel_dudt": pairs["sym"]}
    flops = {k: pass_pairs[k] * FLOP_PER_PAIR[k] for k in pass_pairs}
    dom = max(pass_pairs, key=lambda k: pass_ms[k])
    achieved = flops[dom] / (pass_ms[dom] * 1e-3) / 1e12
    traffic, traffic_src, fp32x = None, None, None
    for rnd in ("r02", "r01"):  # the newest committed ncu capture of the same kernels (c4)
        fn = os.path.join(ROOT, "profiles", rnd, "ncu_fp32.json")
        try:
            with open(fn) as f:
                px = json.load(f)["passes"]
        except Exception:
            continue
        if args.config == "c4" and dom in px:
            traffic = px[dom]["dram_bytes"]
            traffic_src = os.path.relpath(fn, ROOT) + " (dram__bytes_read+write, one launch)"
            fp32x = {k: {"executed_tflops": round(v["executed_tflops"], 3),
                         "frac_of_peak": round(v["frac_of_peak_at_max_clock"], 4),
                         "useful_tflops": round(flops[k] / (pass_ms[k] * 1e-3) / 1e12, 3) if k in flops else None}
                     for k, v in px.items()}
            fp32x["source"] = os.path.relpath(fn, ROOT)
        break
    if traffic is None:
        try:  # round 1's capture
            with open(os.path.join(ROOT, "profiles", "r01", "ncu_traffic.json")) as f:
                tk = json.load(f)["kernels"].get(dom)
            if tk and args.config == "c4" and _DOM_KERNEL.get(dom, "?") in tk["kernel"]:
                traffic = tk["dram_bytes"]
                traffic_src = "profiles/r01/ncu_traffic.json (dram__bytes_read+write, one launch)"
        except Exception:
            pass
    useful_tf = sum(flops.values()) / (ms_step * 1e-3) / 1e12

    # e2e through the public API with host buffers (pinned), H2D + D2H inside the timed region
    e2e = None
    try:
        host = {k: torch.from_numpy(np.ascontiguousarray(parts[k])).pin_memory()
                for k in Particles.IN_F32 + ("species", "id")}
        outk = ["ax", "ay", "az", "ahx", "ahy", "ahz", "dudt", "perm"]
        hout = {k: torch.empty(p.n, dtype=getattr(p, k).dtype).pin_memory() for k in outk}
        bi = sum(t.numel() * t.element_size() for t in host.values())
        bo = sum(t.numel() * t.element_size() for t in hout.values())
        # pipelined through the public API: two device particle sets; while step k computes on
        # `stream`, step k+1's inputs go up on one copy stream and step k-1's results come down
        # on another (PCIe is full duplex); every step still copies its inputs in and its
        # results out
        sets = [p, Particles(p.n, dev, outputs="forces")]
        hout2 = [hout, {k: torch.empty(p.n, dtype=getattr(p, k).dtype).pin_memory() for k in outk}]
        h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_done = [torch.cuda.Event(), torch.cuda.Event()]
        ev_grav = [torch.cuda.Event(), torch.cuda.Event()]
        ev_out = [torch.cuda.Event(), torch.cuda.Event()]
        early = ["perm", "ax", "ay", "az"]  # final once the gravity pass is done

        def run_e2e(nsteps):
            h2d.wait_stream(stream)
            with torch.cuda.stream(h2d):
                sets[0].load(host, non_blocking=True)
            ev_in[0].record(h2d)
            for k in range(nsteps):
                b = k % 2
                stream.wait_event(ev_in[b])
                if k >= 2:
                    stream.wait_event(ev_out[b])  # step k-2's results of this set are down
                step(False, sets[b], grav_done=ev_grav[b])
                ev_done[b].record(stream)
                if k + 1 < nsteps:
                    nb = (k + 1) % 2
                    if k >= 1:
                        h2d.wait_event(ev_done[nb])  # step k-1 is done with that set's inputs
                    with torch.cuda.stream(h2d):
                        sets[nb].load(host, non_blocking=True)
                    ev_in[nb].record(h2d)
                # the gravity results while the hydro passes run, the rest after the step
                d2h.wait_event(ev_grav[b])
                with torch.cuda.stream(d2h):
                    for key in early:
                        hout2[b][key].copy_(getattr(sets[b], key), non_blocking=True)
                d2h.wait_event(ev_done[b])
                with torch.cuda.stream(d2h):
                    for key in outk:
                        if key not in early:
                            hout2[b][key].copy_(getattr(sets[b], key), non_blocking=True)
                ev_out[b].record(d2h)
            stream.wait_stream(d2h)

        run_e2e(2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_e2e(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / args.steps
        e2e = {"value": pair_int * world / (ems * 1e-3), "unit": "pair interactions/s", "ms_per_step": ems,
               "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
               "overlap": "H2D of step k+1 and D2H of step k-1 on two copy streams during step k; "
                          "the gravity results and perm of step k go down while its hydro passes run"}
    except Exception as ex:  # pragma: no cover
        e2e = {"error": str(ex)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        pr, secs, desc, _ = oracle_sample(parts, params)
        cpu = {"value": pr / secs, "unit": "pair interactions/s", "cores": oracle.num_threads(), "kind": "oracle",
               "sample": desc, "seconds": secs, "cpu": _cpu_model(), "seconds_1core_config1": oracle_1core_c1()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pair interactions/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(_config(args, parts), parallelism="replicas" if world > 1 else "single GPU",
                           generator_s=round(gen_s, 1)),
            "pass_ms": {k: round(v, 4) for k, v in pass_ms.items()},
            "substep_ms": ms_step,
            "pairs": pairs, "pair_interactions_per_step": pair_int,
            "useful_fp32_tflops": useful_tf, "useful_fp32_frac_of_peak": useful_tf / peak_tf,
            "fp32_executed": fp32x,
            "fp32_pct_executed": (100 * fp32x[dom]["frac_of_peak"]) if fp32x and dom in fp32x else None,
            "roofline": {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_basis": f"{n_sm} SMs x 128 FP32 lanes x 2 x {f_max:.0f} MHz (sm_max_mhz, MEASURED_PEAKS.json)"},
            "clocks": clk.summary(),
            "e2e": e2e,
            "gpu_launches": int(launches),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
