#!/usr/bin/env python3
"""Long free-running physics check on the GPU (not a bench, not a parity test):
python tools/long_run.py WORKLOAD STEPS EVERY OUT.json

Runs the workload for STEPS steps from its seeded synthetic start, calling
pic_diagnostics every EVERY steps (and at the step after, so the continuity
residual of the deposit is measured), and writes the time series: total
energy (field + kinetic) and its drift, charge, max |div B|, Gauss residual
and its drift from the first call, continuity residual.  The charge-conserving
deposit keeps the Gauss drift at rounding level, div B stays at rounding
level, and in a thermal plasma the total energy drifts only slowly (finite
grid heating); DESIGN.md sec. 10 states the expectations."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1608_01009_b200 as pkg  # noqa: E402
from synth import gen_particles, get_config  # noqa: E402


def main():
    name, steps, every, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    wl = get_config(name)
    sim = pkg.simulation_from_workload(wl)
    for s, (P, ids) in enumerate(gen_particles(wl)):
        sim.set_particles(s, P, ids)
    if wl.laser:   # the open laser box starts with the incident wave in the vacuum
        sim.laser_preload()
    rows = []
    t0 = time.perf_counter()
    done = 0
    while done <= steps:
        d0 = sim.diagnostics()
        sim.step(1)
        d1 = sim.diagnostics()   # at n+1: its continuity residual covers the deposit of step n
        ke = sum(d1["kinetic_energy"])
        rows.append({"step": d1["step"], "field_energy": d1["field_energy"], "kinetic_energy": ke,
                     "total_energy": d1["field_energy"] + ke, "charge": d1["charge"],
                     "max_div_b": d1["max_div_b"], "max_gauss": d1["max_gauss"],
                     "max_gauss_drift": d1["max_gauss_drift"], "max_continuity": d1["max_continuity"]})
        del d0
        done += 1
        if done > steps:
            break
        n = min(every - 1, steps - done + 1)
        if n > 0:
            sim.step(n)
            done += n
    torch.cuda.synchronize()
    e0 = rows[0]["total_energy"]
    res = {"workload": name, "steps": steps, "every": every, "particles": wl.n_particles,
           "wall_s": time.perf_counter() - t0,
           "max_rel_energy_drift": max(abs(r["total_energy"] - e0) / abs(e0) for r in rows),
           "max_div_b": max(r["max_div_b"] for r in rows),
           "max_gauss_drift": max(r["max_gauss_drift"] for r in rows),
           "max_continuity": max(r["max_continuity"] for r in rows),
           "series": rows}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "series"}))
    sim.close()


if __name__ == "__main__":
    main()
