#!/usr/bin/env python3
"""Shared-memory wavefronts per SASS opcode from an ncu report's source page:
python tools/ncu_smem.py report.ncu-rep  (actual vs ideal wavefronts, by opcode)"""
import csv
import subprocess
import sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(lambda: [0, 0, 0, 0])
tot = [0, 0]
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    try:
        wf = float(r[ix["L1 Wavefronts Shared"]] or 0)
        ideal = float(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
        n = float(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    if wf == 0:
        continue
    op = r[ix["Source"]].split()[0]
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    a = agg[op]
    a[0] += wf; a[1] += ideal; a[2] += n; a[3] += 1
    tot[0] += wf; tot[1] += ideal
print(f"total shared wavefronts {tot[0]:.4g}  ideal {tot[1]:.4g}")
for op, (wf, ideal, n, k) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{op:28s} wf {wf:12.4g} ({100*wf/tot[0]:5.1f}%)  ideal {ideal:12.4g}  inst {n:12.4g}  wf/inst {wf/max(n,1):5.2f}  sites {k}")
