#!/usr/bin/env python3
"""Split of the end-to-end path (bench.py's e2e) on one workload: pinned host
-> pic_set_particles (H2D + validation + sort), pic_step(K), pic_get_particles
(D2H), each timed with the host clock around synchronous ABI calls, plus the
H2D / D2H bandwidth of one plain cudaMemcpy of the same bytes.
    python tools/e2e_split.py [WORKLOAD] [K]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1608_01009_b200 as pkg  # noqa: E402
from bench import pinned_copy  # noqa: E402
from synth import gen_particles, get_config  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    wl = get_config(name)
    parts = gen_particles(wl)
    pinned = [pinned_copy(P, ids) for P, ids in parts]
    outs = [pinned_copy(np.empty_like(P), np.empty_like(ids)) for P, ids in parts]
    sim = pkg.simulation_from_workload(wl, capacity_factor=1.0)
    for s, (_, _, Pn, In) in enumerate(pinned):
        sim.set_particles(s, Pn, In)
    sim.step(3)
    torch.cuda.synchronize()
    nbytes = sum(P.nbytes + i.nbytes for P, i in parts)
    for rep in range(2):
        t0 = time.perf_counter()
        for s, (_, _, Pn, In) in enumerate(pinned):
            sim.set_particles(s, Pn, In)
        t1 = time.perf_counter()
        sim.step(K)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        for s in range(len(parts)):
            sim.get_particles(s, out=outs[s][2:])
        t3 = time.perf_counter()
        print(f"{name} K={K}: set_particles {1e3 * (t1 - t0):.1f} ms ({nbytes / (t1 - t0) / 1e9:.1f} GB/s incl. sort), "
              f"steps {1e3 * (t2 - t1):.1f} ms, get_particles {1e3 * (t3 - t2):.1f} ms "
              f"({nbytes / (t3 - t2) / 1e9:.1f} GB/s); e2e {sum(p.shape[1] for p, _ in parts) * K / (t3 - t0) / 1e9:.2f} G upd/s",
              flush=True)
    # plain copies of the same bytes
    dev = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    host = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(host, non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        host.copy_(dev, non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
    print(f"plain cudaMemcpy of {nbytes / 1e9:.2f} GB: H2D {nbytes / (t1 - t0) / 1e9:.1f} GB/s, "
          f"D2H {nbytes / (t2 - t1) / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
