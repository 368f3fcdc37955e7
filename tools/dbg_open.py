#!/usr/bin/env python3
"""Per-array diagnosis of the open-z laser case (T_laser) on the GPU: for the
first steps, teacher-forced from the oracle, prints max |ref| and max |GPU -
ref| of every field component and particle set (python tools/dbg_open.py)."""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1608_01009_b200 as pic
from oracle import oracle as O
from synth import gen_particles, get_config
from tests.test_gpu_open import _oracle, _L
from tests.helpers import by_id
wl = get_config("T_laser")
parts = gen_particles(wl)
orc = _oracle(O, wl, parts); orc.laser_preload()
sim = pic.simulation_from_workload(wl)
for step in range(4):
    sim.set_fields(orc.F[:6].copy())
    for s in range(2): sim.set_particles(s, orc.P[s], orc.ids[s])
    orc.step(1); sim.step(1)
    G = sim.get_fields()
    names = "Ex Ey Ez Bx By Bz Jx Jy Jz".split()
    for c in range(9):
        d = np.abs(G[c]-orc.F[c]); m = np.abs(orc.F[c]).max()
        k = np.unravel_index(np.argmax(d), d.shape)
        print(step, names[c], "max|ref| %.3e max|d| %.3e at %s" % (m, d.max(), k))
    for s in range(2):
        gP, gi = by_id(*sim.get_particles(s)); rP, ri = by_id(orc.P[s], orc.ids[s])
        print(step, "species", s, gP.shape, rP.shape, "dpos %.3e du %.3e umax %.3e" % (np.abs(gP[:3]-rP[:3]).max(), np.abs(gP[3:]-rP[3:]).max(), np.abs(rP[3:]).max()))
