#!/usr/bin/env python3
"""Benchmark of the fp64 PIC step (BASELINE.json metric: particle updates/s,
ns/particle/step, % HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2]
                    [--impl ours|reference] [--no-e2e] [--no-cpu-baseline]

A "step" is one PIC time step of the whole hot path (SURVEY.md sec. 8a:
sort every K steps, fused gather/push/deposit, J fold, Yee update) over the
workload's synthetic particles.  At N=1 the default workload is C3 =
BASELINE.json configs[2], the largest single-GPU configuration (128^3, 25 e +
25 p per cell = 104.9M particles in one fused launch per step; its particle
state, 5.9 GB, is far larger than the 126 MB L2, so no explicit L2 flush);
at N>1 it is C4 (weak scaling).  C1, C2, FROZEN and C5_1g via --workload.

--impl reference times the CPU oracle (oracle/, plain serial C) on the same
workload: each step pushes a fixed bounded sample of the particles through
one oracle step; rank 0 only.
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

METRIC = "particle updates/sec (ns/particle/step), fp64, 1/2/4/8 B200; % HBM roofline"
# the paper's own number exists only for its frozen-plasma
# benchmark (40^3, 50 ppc, 1000 steps): KNL optimised 10.75 s for 3.2e9
# particle-steps (Table 6) -- another machine's number, context.
PAPER_KNL_FROZEN = 3.2e9 / 10.75
UNIT = "particle-updates/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# fp64 work of one particle update as the paper counts it: 336 flop (FMA = 2),
# its VTune figure (PAPER.md:190 with Table 6 times) -- a
# different code; reported beside this kernel's own ncu-counted figure
PAPER_FLOP_PER_UPDATE = 336.0


def load_ncu_counts(workload):
    """Per-launch ncu counts of the fused particle kernel for a workload
    (profiles/ncu_particle_traffic.json): DRAM bytes and the executed fp64
    thread instructions (DFMA counted as 2 flop), with the commit and the
    capture they came from.  ncu cannot run inside the timed bench, so these
    are the last capture's numbers, labelled as such."""
    p = os.path.join(ROOT, "profiles", "ncu_particle_traffic.json")
    if not os.path.exists(p):
        return {}, None
    with open(p) as f:
        d = json.load(f)
    return d.get(workload, {}), d.get("_source")


def load_fp64_peak():
    """DFMA peak measured on a B200 by tools/microbench.cu (TFLOP/s)."""
    p = os.path.join(ROOT, "profiles", "r01", "microbench.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["dfma_tflops"]), "measured (profiles/r01/microbench.json dfma_tflops)"
    return 37.2, "datasheet (148 SM x 64 FP64 lanes x 2 x 1.965 GHz), not measured"


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """Samples SM clock and throttle reasons with NVML every ~1 ms."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self.nv = None
            self.err = str(e)
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        reasons = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ helpers

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def reduce_max_over_ranks(v: float) -> float:
    """max of a float over the initialised process group (identity without one)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(v)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum_over_ranks(v: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(v)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    return float(t.item())


# per-plane cost of the static load balance (NEXT-1): time per particle-step
# and per cell-step in particle-step units (B200: 0.055 ns per particle
# (C3 particle kernel + sort), 0.064 ns per cell (C3 field stage))
CELL_COST = 1.2


def slab_split(wl, world):
    """z cut planes of the world ranks: uniform nz/world, or -- for a workload
    whose plasma fills only part of the box (C5) -- pic_balance_slabs on
    particles + CELL_COST x cells per plane."""
    if world == 1 or not wl.plasma_z:
        return [r * (wl.nz // world) for r in range(world)] + [wl.nz]
    import paper_1608_01009_b200 as pkg
    ppc = sum(s.ppc for s in wl.species)
    cost = np.full(wl.nz, CELL_COST * wl.nx * wl.ny)
    cost[wl.plasma_z[0]:wl.plasma_z[1]] += ppc * wl.nx * wl.ny
    return pkg.balance_slabs(wl.nz, world, wl.supercell, max(4, wl.supercell), cost)


def occupied_cells(wl, lo, hi):
    """Cells of the planes [lo, hi) that hold particles (the E/B tile gather
    and the J flush of the particle kernel touch only those)."""
    if wl.plasma_z:
        lo, hi = max(lo, wl.plasma_z[0]), min(hi, wl.plasma_z[1])
    return wl.nx * wl.ny * max(0, hi - lo)


def oracle_grid(O, wl):
    lz = dict(wl.laser) if wl.laser else {}
    return O.Grid(wl.nx, wl.ny, wl.nz, wl.dx, wl.dy, wl.dz, wl.dt, wl.c,
                  [O.Species(s.q, s.m, s.w) for s in wl.species], wl.supercell, wl.sort_every,
                  bc_z=O.BC_OPEN if wl.open_z else O.BC_PERIODIC,
                  laser_e0=lz.get("e0", 0.0), laser_omega=lz.get("omega", 0.0),
                  laser_ramp=lz.get("ramp", 0.0), laser_t0=lz.get("t0", 0.0),
                  laser_pol=tuple(lz.get("pol", (1.0, 0.0))))


def pinned_copy(P, ids):
    import torch
    tp = torch.empty(P.shape, dtype=torch.float64, pin_memory=True)
    tp.numpy()[:] = P
    ti = torch.empty(ids.shape, dtype=torch.int64, pin_memory=True)
    ti.numpy().view(np.uint64)[:] = ids
    return tp, ti, tp.numpy(), ti.numpy().view(np.uint64)


def oracle_sample_rate(wl, parts, target_s=10.0, max_particles=None):
    """Time the oracle as it stands (single thread) on a bounded sample:
    full oracle steps of the workload when one fits in target_s, else a
    contiguous particle sample pushed through one oracle step."""
    from oracle import oracle as O
    O.build()
    g = oracle_grid(O, wl)
    sub = []
    n_tot = sum(p.shape[1] for p, _ in parts)
    if max_particles is None:   # ~0.4 us per particle-step single threaded: bound the sample
        max_particles = int(target_s * 1.0e6)
    frac = min(1.0, max_particles / n_tot)
    for P, ids in parts:
        k = max(1, int(P.shape[1] * frac))
        sub.append((P[:, :k].copy(), ids[:k].copy()))
    orc = O.Oracle(g, particles=sub)
    if wl.laser:
        orc.laser_preload()
    n_sample = sum(p.shape[1] for p, _ in sub)
    t0 = time.perf_counter()
    steps = 0
    while True:
        orc.step(1)
        steps += 1
        if time.perf_counter() - t0 >= target_s:
            break
    dt = time.perf_counter() - t0
    return n_sample * steps / dt, n_sample, steps, dt


def host_info():
    """The host the oracle ran on: logical CPUs and the CPU model."""
    import platform
    host = {"nproc": os.cpu_count(), "cpu": platform.processor() or platform.machine(), "threads_used": 1}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    host["cpu"] = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return host


def data_pipe_roof(ncu, launch_ms, sm_mhz):
    """The binding resource of the fused particle kernel:
    the SM's L1/shared-memory data pipe, one 128-byte wavefront per SM clock
    for every LDS, STS, ATOMS (a read and a write wavefront), LDGSTS fill,
    global load/store and local spill.  achieved = the ncu-counted wavefronts
    of one launch (profiles/ncu_particle_traffic.json, the commit it was
    captured at) over this run's launch time; peak = 148 SMs x the SM clock
    sampled under load."""
    w = ncu.get("lsu_wavefronts_per_launch")
    if not w or not sm_mhz:
        return None
    peak = 148 * sm_mhz * 1e6
    achieved = w / (launch_ms * 1e-3)
    return {"unit": "wavefronts/s", "achieved": achieved, "peak": peak, "frac": achieved / peak,
            "wavefronts_per_launch": w, "source": f"ncu l1tex__data_pipe_lsu_wavefronts.sum at commit "
                                                  f"{ncu.get('commit', '?')}; peak = 148 SM x {sm_mhz:.0f} MHz"}


def fp64_roof(rate_per_gpu, flop_upd, ncu, peak, peak_src):
    """The FP64 roof of SURVEY.md sec. 8d from this kernel's own counted work
    per update (ncu opcode mix of the captured launch, null if none), with
    the paper's 336 flop/update alongside as a labelled figure."""
    out = {"peak_tflops": peak, "peak_source": peak_src,
           "paper_flop_per_update": PAPER_FLOP_PER_UPDATE,
           "paper_frac": rate_per_gpu * PAPER_FLOP_PER_UPDATE / 1e12 / peak}
    if flop_upd:
        out.update({"flop_per_update": flop_upd,
                    "flop_source": f"ncu sm__sass_thread_inst_executed_op_d{{fma,add,mul}}_pred_on "
                                   f"(DFMA = 2 flop) of the particle kernel at commit {ncu.get('commit', '?')}; "
                                   f"the sort and field kernels' few fp64 operations are not included",
                    "achieved_tflops": rate_per_gpu * flop_upd / 1e12,
                    "frac": rate_per_gpu * flop_upd / 1e12 / peak})
    else:
        out.update({"flop_per_update": None, "achieved_tflops": None, "frac": None})
    return out


# ------------------------------------------------------------------ arms

def run_reference(args, wl, rank, world):
    if rank != 0:
        return
    from synth import gen_particles
    n_sample = args.ref_sample
    # a bounded sample: generate only the first z planes that hold it (the
    # same distribution as the whole workload; C3 would be 105M particles)
    ppc = sum(s.ppc for s in wl.species)
    z0 = wl.plasma_z[0] if wl.plasma_z else 0
    planes = min(wl.nz - z0, max(1, -(-n_sample // (ppc * wl.nx * wl.ny))))
    parts = gen_particles(wl, z_lo=z0, z_hi=z0 + planes)
    from oracle import oracle as O
    O.build()
    g = oracle_grid(O, wl)
    sub = []
    for P, ids in parts:
        k = min(P.shape[1], max(1, n_sample // len(parts)))
        sub.append((P[:, :k].copy(), ids[:k].copy()))
    orc = O.Oracle(g, particles=sub)
    if wl.laser:
        orc.laser_preload()
    ns = sum(p.shape[1] for p, _ in sub)
    for _ in range(args.warmup):
        orc.step(1)
    t0 = time.perf_counter()
    orc.step(args.steps)
    dt = time.perf_counter() - t0
    v = ns * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "ns_per_particle_step": 1e9 / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": wl_config(wl, world, slab_split(wl, world)),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"first {ns} particles of {wl.name} (of {wl.n_particles}) "
                                   f"through full oracle steps (fields on the whole grid), "
                                   f"single thread",
                         "host": host_info()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def wl_config(wl, world, split=None):
    c = {"workload": wl.name, "grid": [wl.nx, wl.ny, wl.nz],
         "particles": wl.n_particles, "species": len(wl.species),
         "ppc": sum(s.ppc for s in wl.species), "sort_every": wl.sort_every,
         "supercell": wl.supercell, "dt": wl.dt,
         "parallelism": f"z-slabs x{world}" if world > 1 else "single GPU",
         "l2": "inputs larger than L2 (particle state > 126 MB), no flush"}
    if wl.open_z:
        lz = dict(wl.laser)
        c["boundary"] = (f"open z (first-order Mur), laser e0={lz['e0']:.4f} omega={lz['omega']:.4f} "
                         f"t0={lz['t0']} ramp={lz['ramp']}, plasma z in {list(wl.plasma_z)}")
    if split is not None and world > 1:
        c["slabs"] = list(split)
    return c


def run_ours(args, wl, rank, world, local):
    import torch

    import paper_1608_01009_b200 as pkg
    from synth import gen_particles

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    split = slab_split(wl, world)
    slab = (split[rank], split[rank + 1])
    if world > 1:
        parts = gen_particles(wl, rank=rank, z_lo=slab[0], z_hi=slab[1])
    else:
        parts = gen_particles(wl)
    n_local = sum(p.shape[1] for p, _ in parts)

    def new_sim(flags=0):
        # every context gets its own NCCL communicator, so a fresh unique id
        # (an id bootstraps exactly one ncclCommInitRank); collective over ranks
        nccl_id = None
        if world > 1:
            nccl_id = pkg.broadcast_nccl_id(pkg.nccl_unique_id() if rank == 0 else bytes(128))
        return pkg.simulation_from_workload(wl, capacity_factor=1.0, flags=flags, rank=rank,
                                            nranks=world, nccl_id=nccl_id, slab=slab)

    def load(sim, ps):
        for s, (P, ids) in enumerate(ps):
            sim.set_particles(s, P, ids)
        if wl.laser and sim.step_index() == 0:
            sim.laser_preload()   # C5: the wave that entered through z = 0 before t = 0

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # ---------------- device-resident timed region (value)
    sim = new_sim()
    load(sim, parts)
    sim.step(args.warmup)
    sim.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(sim.stream)
        sim.step(args.steps)
        e1.record(sim.stream)
        torch.cuda.synchronize()
        barrier()
    t_ms = reduce_max_over_ranks(e0.elapsed_time(e1))
    launches = sim.launch_count()
    n_total = reduce_sum_over_ranks(float(n_local))
    value = n_total * args.steps / (t_ms * 1e-3)
    sim.close()
    del sim
    torch.cuda.empty_cache()

    # ---------------- profiled pass: per-stage CUDA events around each launch
    psim = new_sim(pkg.FLAG_PROFILE)
    load(psim, parts)
    psim.step(args.warmup)
    psim.stage_times()
    psim.step(args.steps)
    st = psim.stage_times()
    psim.close()
    del psim
    torch.cuda.empty_cache()
    # per-rank stage split (N > 1): the exchange on its own stream, overlapped
    # with the interior supercell layers, and the particle stage of every rank
    by_rank = None
    if world > 1:
        import torch.distributed as dist
        mine = {k: st[k] / args.steps for k in ("sort", "particle", "field", "exchange")}
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        by_rank = {k: [g[k] for g in gathered] for k in mine}
    ppc_cells = occupied_cells(wl, slab[0], slab[1])
    n_launch = max(st["particle_launches"], 1)
    per_step_launches = n_launch / args.steps   # species per launch: 1, or all of them (sparse box)
    # algorithmic bytes of one launch: x, u read + write (96 B) of its particles,
    # E/B tile gather (48 B) + J write (24 B) of the occupied cells once per launch
    per_launch_bytes = (n_local * 96.0) / per_step_launches + ppc_cells * 72.0
    alg_bytes_total = per_launch_bytes * per_step_launches
    per_launch_ms = st["particle"] / n_launch
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
    peak, peak_src = load_peaks()
    fp64_peak, fp64_src = load_fp64_peak()
    n_cells_local = wl.nx * wl.ny * (slab[1] - slab[0])
    ncu, ncu_src = load_ncu_counts(wl.name)
    traffic = ncu.get("bytes_per_launch")
    traffic_src = (f"ncu --set full of one launch at commit {ncu.get('commit', '?')} "
                   f"({ncu.get('capture', ncu_src)}), not measured in this run") if traffic else None
    # this kernel's own fp64 work per update (ncu opcode counts of the captured
    # launch: 2 DFMA + DADD + DMUL thread instructions over its particles)
    flop_upd = ncu.get("fp64_flop_per_update")
    step_ms_prof = (st["sort"] + st["particle"] + st["field"] + st["exchange"]) / args.steps

    # ---------------- e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        pinned = [pinned_copy(P, ids) for P, ids in parts]
        outs = [pinned_copy(np.empty_like(P), np.empty_like(ids)) for P, ids in parts]   # pinned results
        esim = new_sim()
        load(esim, [(Pn, In) for _, _, Pn, In in pinned])
        esim.step(args.warmup)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s, (_, _, Pn, In) in enumerate(pinned):
            esim.set_particles(s, Pn, In)
        esim.step(args.steps)
        for s in range(len(parts)):
            esim.get_particles(s, out=outs[s][2:])
        torch.cuda.synchronize()
        barrier()
        te = reduce_max_over_ranks(time.perf_counter() - t0)
        esim.close()
        bytes_io = n_local * 56.0
        e2e = {"value": n_total * args.steps / te, "unit": UNIT,
               "h2d_bytes_per_step": bytes_io / args.steps, "d2h_bytes_per_step": bytes_io / args.steps,
               "mode": "pinned host -> pic_set_particles (incl. sort) -> pic_step(K) -> "
                       "pic_get_particles -> host, wall clock, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, ns, nsteps, dt = oracle_sample_rate(wl, parts, target_s=args.cpu_seconds,
                                               max_particles=args.cpu_max_particles)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{nsteps} oracle step(s) over {ns} of {wl.n_particles} particles of "
                         f"{wl.name} (whole grid), {dt:.1f} s, single thread",
               "host": host_info()}

    csum = clk.summary()
    clk_mhz_hint = csum.get("sm_mhz") or csum.get("sm_max_mhz")
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "ns_per_particle_step": 1e9 / value, "value_per_gpu": value / world,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": value / PAPER_KNL_FROZEN if wl.name == "FROZEN" else None,
            "dtype": "f64",
            "data": "synthetic (seeded numpy PCG64, DESIGN.md sec. 6)",
            "config": wl_config(wl, world, split),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": "particle (gather+Boris+VB deposit)",
                         "alg_bytes_per_launch": per_launch_bytes,
                         "avg_launch_ms": per_launch_ms, "peak_source": peak_src,
                         "timing": "CUDA events around every particle-kernel launch on the "
                                   "library stream, profiled pass of the same K steps",
                         "step_share": st["particle"] / max(1e-9, step_ms_prof * args.steps),
                         "stage_ms_per_step": {k: st[k] / args.steps for k in
                                               ("sort", "particle", "field", "exchange")},
                         # whole step: particle kernel bytes + sort (112 B/particle per
                         # sort) + the Yee update (read E, B, J, write E, B: 120 B/cell)
                         "whole_step_frac": (alg_bytes_total + n_local * 112.0 / max(wl.sort_every, 1)
                                             + n_cells_local * 120.0)
                         / (t_ms * 1e-3 / args.steps) / 1e9 / peak,
                         # the second roof (report both fractions)
                         "fp64": fp64_roof(value / world, flop_upd, ncu, fp64_peak, fp64_src),
                         "data_pipe": data_pipe_roof(ncu, per_launch_ms, clk_mhz_hint)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "stage_ms_per_step_by_rank": by_rank,
            "clocks": csum,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def cpu_baseline_all(path, seconds):
    """The cpu_baseline leg over every workload (no GPU): the oracle as it
    stands, one thread, on bounded samples (SURVEY.md sec. 8d oracle timing);
    C1, C2 and FROZEN whole, the larger ones a particle sample over the whole
    grid.  Writes a JSON file and prints one line per workload."""
    import platform
    from synth import gen_particles, get_config
    rows = []
    for name in ("C1", "C2", "C3", "C4", "C5_1g", "FROZEN"):
        wl = get_config(name)
        parts = gen_particles(wl)
        v, ns, nsteps, dt = oracle_sample_rate(wl, parts, target_s=seconds)
        rows.append({"workload": name, "particles": wl.n_particles, "sample_particles": ns, "steps": nsteps,
                     "seconds": dt, "updates_per_s": v, "ns_per_particle_step": 1e9 / v,
                     "whole": ns == wl.n_particles})
        print(json.dumps(rows[-1]), flush=True)
    host = host_info()
    with open(path, "w") as f:
        json.dump({"host": host, "target_s": seconds, "rows": rows}, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-max-particles", type=int, default=None)
    ap.add_argument("--ref-sample", type=int, default=50_000)
    ap.add_argument("--supercell", type=int, default=None, help="override S (tools/sweep.py)")
    ap.add_argument("--sort-every", type=int, default=None, help="override K (tools/sweep.py)")
    ap.add_argument("--cpu-baseline-all", default=None, metavar="OUT.json",
                    help="only time the oracle (cpu_baseline leg) on every workload; no GPU")
    args = ap.parse_args()
    if args.cpu_baseline_all:
        cpu_baseline_all(args.cpu_baseline_all, args.cpu_seconds)
        return
    assert args.warmup >= 3 or args.impl == "reference", "W >= 3 warm-up steps"
    rank, world, local = dist_env()
    from synth import get_config
    # N = 1: the largest single-GPU configuration (BASELINE.json configs[2]);
    # N > 1: the weak-scaling slab run (configs[3])
    name = args.workload or ("C3" if world == 1 else "C4")
    wl = get_config(name).for_ranks(world)
    if args.supercell:
        wl = wl.with_(supercell=args.supercell)
    if args.sort_every is not None:
        wl = wl.with_(sort_every=args.sort_every)
    if args.impl == "reference":
        run_reference(args, wl, rank, world)
    else:
        run_ours(args, wl, rank, world, local)


if __name__ == "__main__":
    main()
