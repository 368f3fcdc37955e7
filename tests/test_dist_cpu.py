"""World-size-2 gloo tests of the host side of the z-slab (N > 1) path on
CPU: NCCL id distribution through torch.distributed, per-rank slab
configuration (pure sizing calls, no GPU), and bench.py's max-over-ranks
timing / aggregation."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    import ctypes as C
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1608_01009_b200 as pkg
    from synth import get_config

    import bench

    uid = None
    if rank == 0:
        try:
            uid = pkg.nccl_unique_id()
        except Exception:
            uid = os.urandom(128)
    uid = pkg.broadcast_nccl_id(uid if uid is not None else bytes(128))
    wl = get_config("C4").for_ranks(world)
    cfg = pkg.workload_config(wl, rank=rank, nranks=world, nccl_id=uid)
    nb = C.c_size_t(0)
    rc = pkg.lib().pic_workspace_size(C.byref(cfg), C.byref(nb))
    # C5 (NEXT-1): balanced unequal slabs of an open box, ring cut at the faces
    wl5 = get_config("C5")
    split = bench.slab_split(wl5, world)
    cfg5 = pkg.workload_config(wl5, rank=rank, nranks=world, nccl_id=uid,
                               slab=(split[rank], split[rank + 1]))
    rc5 = pkg.lib().pic_workspace_size(C.byref(cfg5), C.byref(C.c_size_t(0)))
    results[(rank, "c5")] = (list(split), rc5, int(cfg5.slab_lo), int(cfg5.slab_hi), int(cfg5.bc_z))
    t_max = bench.reduce_max_over_ranks(float(rank + 1))
    n_tot = bench.reduce_sum_over_ranks(float(10 * (rank + 1)))
    results[rank] = (uid, rc, nb.value, int(cfg.capacity[0]), int(cfg.nz), t_max, n_tot)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_slab_setup_over_gloo():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, results)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    r0, r1 = results[0], results[1]
    assert r0[0] == r1[0] and len(r0[0]) == 128          # same NCCL id on both ranks
    assert r0[1] == 0 and r1[1] == 0                      # valid slab configs
    assert r0[2] == r1[2] > 0                             # identical slab workspace
    per_rank = 256 * 256 * 128 * 32
    assert r0[3] == r1[3] >= int(1.1 * per_rank) - 1      # 10% migration headroom
    assert r0[4] == 256                                   # global nz = 128 per rank
    assert r0[5] == r1[5] == 2.0                          # max over ranks
    assert r0[6] == r1[6] == 30.0                         # sum over ranks
    c0, c1 = results[(0, "c5")], results[(1, "c5")]
    assert c0[0] == c1[0] and c0[0][0] == 0 and c0[0][-1] == 1024
    assert c0[1] == c1[1] == 0 and c0[4] == 1              # valid open-z configs
    assert (c0[2], c0[3]) == (0, c0[0][1]) and (c1[2], c1[3]) == (c0[0][1], 1024)
    assert 600 < c0[0][1] < 700                           # the cut falls inside the slab
