#!/usr/bin/env python3
"""supercell size S and sort interval K sweep with a per-stage
breakdown in the shape of the paper's Tables 5/6.  Prints a
markdown table; run under gpurun:  python tools/sweep.py C3 > profiles/.../sweep.md"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(wl, steps, extra):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", wl, "--steps", str(steps),
           "--warmup", "5", "--no-cpu-baseline", "--no-e2e"] + extra
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1200).stdout.strip().splitlines()
    return json.loads(out[-1])


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    print(f"# {wl}: supercell S / sort interval K sweep ({steps} steps)\n")
    print("| S | K | G upd/s | ns/particle/step | particle ms/step | sort ms/step | field ms/step | kernel HBM frac |")
    print("|---|---|---|---|---|---|---|---|")
    for S in (4, 2):
        for K in (5, 10, 20, 40):
            d = run(wl, steps, ["--supercell", str(S), "--sort-every", str(K)])
            st = d["roofline"]["stage_ms_per_step"]
            print(f"| {S} | {K} | {d['value'] / 1e9:.2f} | {d['ns_per_particle_step']:.4f} | "
                  f"{st['particle']:.4f} | {st['sort']:.4f} | {st['field']:.4f} | {d['roofline']['frac']:.3f} |",
                  flush=True)


if __name__ == "__main__":
    main()
