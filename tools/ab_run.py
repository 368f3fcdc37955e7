#!/usr/bin/env python3
"""A/B timing of the installed libpic.so on one workload (tools/ab.sh):
python tools/ab_run.py WORKLOAD STEPS -> one JSON line (G updates/s, particle ms per launch, stages)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1608_01009_b200 as pkg  # noqa: E402
from synth import gen_particles, get_config  # noqa: E402


def main():
    # WORKLOAD[:hH][:kK]  (halo / sort interval overrides, e.g. C3:h2:k40)
    spec, steps = sys.argv[1], int(sys.argv[2])
    name, *mods = spec.split(":")
    wl = get_config(name)
    for m in mods:
        if m[0] == "h":
            wl = wl.with_(halo=int(m[1:]))
        elif m[0] == "k":
            wl = wl.with_(sort_every=int(m[1:]))
        elif m[0] == "s":
            wl = wl.with_(supercell=int(m[1:]))
    parts = gen_particles(wl)
    n = sum(p.shape[1] for p, _ in parts)
    out = {"workload": spec}
    for flags in (0, pkg.FLAG_PROFILE):
        sim = pkg.simulation_from_workload(wl, capacity_factor=1.0, flags=flags)
        for s, (P, ids) in enumerate(parts):
            sim.set_particles(s, P, ids)
        sim.step(5)
        if flags:
            sim.stage_times()
            sim.step(steps)
            st = sim.stage_times()
            out["particle_ms_launch"] = round(st["particle"] / max(st["particle_launches"], 1), 5)
            out["stage_ms_step"] = {k: round(st[k] / steps, 4) for k in ("sort", "particle", "field")}
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(sim.stream)
            sim.step(steps)
            e1.record(sim.stream)
            torch.cuda.synchronize()
            out["gups"] = round(n * steps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 3)
        sim.close()
        del sim
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
