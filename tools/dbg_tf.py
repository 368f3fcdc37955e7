import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1608_01009_b200 as pkg
from synth import get_config, gen_particles
from oracle import oracle as O
wl = get_config(sys.argv[1] if len(sys.argv) > 1 else "C1")
parts = gen_particles(wl)
g = O.Grid(wl.nx, wl.ny, wl.nz, wl.dx, wl.dy, wl.dz, wl.dt, wl.c, [O.Species(s.q, s.m, s.w) for s in wl.species], wl.supercell, wl.sort_every)
orc = O.Oracle(g, particles=[(p.copy(), i.copy()) for p, i in parts])
sim = pkg.simulation_from_workload(wl)
for step in range(int(sys.argv[2]) if len(sys.argv) > 2 else 10):
    sim.set_fields(orc.F[:6].copy())
    for s in range(len(wl.species)):
        sim.set_particles(s, orc.P[s], orc.ids[s])
    orc.step(1)
    try:
        sim.step(1)
    except Exception as e:
        print("step", step, "failed:", e); raise
    print("step", step, "ok", flush=True)
