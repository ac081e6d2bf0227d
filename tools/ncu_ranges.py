#!/usr/bin/env python
"""Sum an ncu source page (needs -lineinfo, --import-source on) over named line
ranges of one file.  usage: ncu_ranges.py report.ncu-rep file.cuh name:lo-hi ..."""
import csv
import io
import os
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for spec in sys.argv[3:]:
    name, span = spec.split(":")
    lo, hi = (int(x) for x in span.split("-"))
    ranges.append((name, lo, hi))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if len(r) > 5 and r[0] == "Line No")
ie, te, ss = (hdr.index(k) for k in ("Instructions Executed", "Thread Instructions Executed",
                                      "Warp Stall Sampling (All Samples)"))
acc = {n: [0.0, 0.0, 0.0] for n, _, _ in ranges}
acc["(other files)"] = [0.0, 0.0, 0.0]
acc["(other lines)"] = [0.0, 0.0, 0.0]
cur = "?"
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = os.path.basename(r[1])
        continue
    if len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
        v = [float(r[ie] or 0), float(r[te] or 0), float(r[ss] or 0)]
        key = "(other files)"
        if cur == fname:
            key = next((n for n, lo, hi in ranges if lo <= int(r[0]) <= hi), "(other lines)")
        for i in range(3):
            acc[key][i] += v[i]
tot = [sum(a[i] for a in acc.values()) for i in range(3)]
print(f"total warp-instr {tot[0]:.3e}")
for n, a in acc.items():
    print(f"{n:16s} warp-instr {a[0]:.3e} ({a[0]/tot[0]*100:5.1f}%)  thr/warp {a[1]/max(a[0],1):5.1f}  "
          f"stall {a[2]/max(tot[2],1)*100:5.1f}%")
