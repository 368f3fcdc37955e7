#!/usr/bin/env python3
"""Aggregate ncu warp-stall samples by CUDA source line (needs -lineinfo):
python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        try:
            agg[(cur, int(r[0]))] = (int(r[4]), int(r[7]), r[1][:90])
        except (ValueError, IndexError):
            pass
tot = sum(v[0] for v in agg.values()) or 1
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{k[0]}:{k[1]}".ljust(26), str(v[0]).rjust(5), "%4.1f%%" % (100 * v[0] / tot), str(v[1]).rjust(9), v[2])
