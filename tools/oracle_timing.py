#!/usr/bin/env python3
"""Times the CPU oracle as it stands (single thread) on each BASELINE workload,
the way bench.py's cpu_baseline does (bounded samples; SURVEY.md sec. 8d
"oracle timing"): python tools/oracle_timing.py OUT.json [seconds]
C1 runs whole; the larger workloads push a contiguous particle sample over
the whole grid (ns/particle/step extrapolated from it)."""
import json
import os
import platform
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from synth import gen_particles, get_config  # noqa: E402


def main():
    out = sys.argv[1]
    target = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
    rows = []
    for name in ("C1", "C2", "C3", "C4", "C5_1g", "FROZEN"):
        wl = get_config(name)
        parts = gen_particles(wl)
        v, ns, nsteps, dt = bench.oracle_sample_rate(wl, parts, target_s=target)
        rows.append({"workload": name, "particles": wl.n_particles, "sample_particles": ns, "steps": nsteps,
                     "seconds": dt, "updates_per_s": v, "ns_per_particle_step": 1e9 / v,
                     "whole": ns == wl.n_particles})
        print(json.dumps(rows[-1]), flush=True)
    host = {"cpu": platform.processor() or platform.machine(), "nproc": os.cpu_count(), "threads_used": 1}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    host["cpu"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    with open(out, "w") as f:
        json.dump({"host": host, "target_s": target, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
