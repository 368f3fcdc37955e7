#!/usr/bin/env python3
"""Warp-level instructions executed per CUDA source line (needs -lineinfo):
python tools/ncu_inst_lines.py report.ncu-rep [top] [per]   (per: divide counts, e.g. by warps of particles)"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
per = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
agg = {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        agg[(cur, int(r[0]))] = (int(r[7]), int(r[4]), r[1].strip()[:88])
    except (ValueError, IndexError):
        pass
tot = sum(v[0] for v in agg.values()) or 1
print(f"total {tot:.4g} warp instructions, {tot / per:.1f} per unit")
for (f, ln), (n, smp, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{f}:{ln}".ljust(26), f"{n / per:8.2f} {100 * n / tot:5.1f}%  smp {smp:5d}  {src}")
