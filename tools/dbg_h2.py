import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1608_01009_b200 as pkg
from synth import gen_particles, get_config
from synth.configs import electron, proton
for S, h, sp in [(2,2,1),(4,2,1),(4,2,2),(4,1,2)]:
    wl = get_config("C1").with_(supercell=S, halo=h, sort_every=5)
    if sp == 2:
        wl = wl.with_(species=(electron(3, 0.3), proton(2, 200.0)))
    parts = gen_particles(wl)
    try:
        sim = pkg.simulation_from_workload(wl, flags=pkg.FLAG_NO_GRAPH)
        for s,(P,ids) in enumerate(parts): sim.set_particles(s,P,ids)
        sim.step(3)
        print(S,h,sp,"ok", flush=True)
    except Exception as e:
        print(S,h,sp,"FAIL",e, flush=True)
        break
