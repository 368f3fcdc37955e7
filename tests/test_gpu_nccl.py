"""Two-rank z-slab step over real NCCL (one process per GPU, torchrun-style
rendezvous on 127.0.0.1): the captured-graph step (NCCL send/recv of the J
ghost planes and migrating particles on the exchange stream, overlapped with
the interior supercell layers; E/B ghost planes) and the uncaptured one,
against the single-domain oracle (P16) and against the in-process slab
group (PIC_FLAG_LOCAL_GROUP) of the same split.  Needs >= 2 visible GPUs;
skipped on the 1-GPU pool (ADVICE runtime.cu:439)."""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEPS = 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload():
    from synth import get_config
    from synth.configs import electron
    # 2 ranks x 16 planes: 4 supercell layers per slab (boundary 0, 3; interior 1, 2)
    return get_config("C1").with_(species=(electron(6, 0.2),), nz=32, sort_every=5)


def _fields(wl):
    rng = np.random.default_rng(23)
    return rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.02


def _rank_main(rank, world, port, outdir, flags):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_1608_01009_b200 as pkg
    from synth import gen_particles
    wl = _workload()
    parts = gen_particles(wl)
    F6 = _fields(wl)
    nzl = wl.nz // world
    uid = pkg.broadcast_nccl_id(pkg.nccl_unique_id() if rank == 0 else bytes(128))
    sim = pkg.simulation_from_workload(wl, rank=rank, nranks=world, nccl_id=uid, flags=flags,
                                       migrate_capacity=4096)
    sim.set_particles(0, *parts[0])
    sim.set_fields(F6[:, rank * nzl:(rank + 1) * nzl].copy())
    for step in range(STEPS):
        sim.step(1)
        P, ids = sim.get_particles(0)
        np.savez(os.path.join(outdir, f"r{rank}_s{step}.npz"), F=sim.get_fields(), P=P, ids=ids)
    st = sim.stage_times() if flags & pkg.FLAG_PROFILE else None
    if st is not None:
        np.save(os.path.join(outdir, f"r{rank}_stage.npy"), np.array([st["exchange"]]))
    sim.close()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def two_gpus():
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (the pool gives one)")


@pytest.mark.parametrize("flags_name", ["graphs", "no_graph_profiled"])
def test_two_rank_nccl_step_matches_oracle_and_local_group(two_gpus, oracle_mod, flags_name):
    import torch
    import torch.multiprocessing as mp
    import paper_1608_01009_b200 as pkg
    from synth import gen_particles
    from tests.helpers import compare_state, field_errs
    flags = 0 if flags_name == "graphs" else (pkg.FLAG_NO_GRAPH | pkg.FLAG_PROFILE)
    wl = _workload()
    with tempfile.TemporaryDirectory() as outdir:
        mp.spawn(_rank_main, args=(2, _free_port(), outdir, flags), nprocs=2, join=True)
        parts = gen_particles(wl)
        F6 = _fields(wl)
        g = oracle_mod.Grid(wl.nx, wl.ny, wl.nz, wl.dx, wl.dy, wl.dz, wl.dt, wl.c,
                            [oracle_mod.Species(s.q, s.m, s.w) for s in wl.species], wl.supercell, wl.sort_every)
        orc = oracle_mod.Oracle(g, particles=[(p.copy(), i.copy()) for p, i in parts])
        orc.F[:6] = F6
        # the same split as an in-process slab group on GPU 0
        stream = torch.cuda.Stream()
        sims = [pkg.Simulation(pkg.workload_config(wl, rank=r, nranks=2, flags=pkg.FLAG_LOCAL_GROUP,
                                                   migrate_capacity=4096), stream=stream) for r in range(2)]
        nzl = wl.nz // 2
        for r, sim in enumerate(sims):
            sim.set_particles(0, *parts[0])
            sim.set_fields(F6[:, r * nzl:(r + 1) * nzl].copy())
        L = (wl.nx * wl.dx, wl.ny * wl.dy, wl.nz * wl.dz)
        for step in range(STEPS):
            orc.step(1)
            pkg.step_group(sims, 1)
            ranks = [np.load(os.path.join(outdir, f"r{r}_s{step}.npz")) for r in range(2)]
            G = np.concatenate([d["F"] for d in ranks], axis=1)
            gP = np.concatenate([d["P"] for d in ranks], axis=1)
            gi = np.concatenate([d["ids"] for d in ranks])
            pe, ue = compare_state(gP, gi, orc.P[0], orc.ids[0], L)
            assert max(field_errs(G, orc.F) + [pe, ue]) <= 1e-11, step
            # NCCL transport == device-to-device transport (up to the order of
            # the fp64 REDG flushes of overlapping tiles)
            Gl = np.concatenate([s.get_fields() for s in sims], axis=1)
            assert max(field_errs(G, Gl)) <= 1e-13, step
            for r, sim in enumerate(sims):
                Pl, il = sim.get_particles(0)
                assert np.array_equal(np.sort(il), np.sort(ranks[r]["ids"])), (step, r)
        if flags:
            exch = [float(np.load(os.path.join(outdir, f"r{r}_stage.npy"))[0]) for r in range(2)]
            assert all(e > 0 for e in exch)
