#!/usr/bin/env python3
"""Minimal driver for profiling: build a Simulation for a workload, load its
particles, run N steps (python tools/run_steps.py C2 5 [flags])."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1608_01009_b200 as pkg  # noqa: E402
from synth import gen_particles, get_config  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    wl = get_config(name)
    parts = gen_particles(wl)
    sim = pkg.simulation_from_workload(wl, flags=flags)
    for s, (P, ids) in enumerate(parts):
        sim.set_particles(s, P, ids)
    t0 = time.perf_counter()
    sim.step(n)
    torch.cuda.synchronize()
    print(f"{name}: {n} steps in {time.perf_counter() - t0:.4f} s")


if __name__ == "__main__":
    main()
