#!/usr/bin/env python
"""Sum an ncu source page (cuda lines) over named line ranges.
usage: ncu_regions.py report.ncu-rep file.cuh name:lo-hi [name:lo-hi ...]"""
import csv, io, os, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
regions = []
for a in sys.argv[3:]:
    n, r = a.split(":"); lo, hi = r.split("-"); regions.append((n, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if len(r) > 5 and r[0] == "Line No")
ie = hdr.index("Instructions Executed"); te = hdr.index("Thread Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
cur = "?"; acc = {n: [0, 0, 0] for n, _, _ in regions}; acc["other"] = [0, 0, 0]; tot = [0, 0, 0]
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = os.path.basename(r[1]); continue
    if len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
        v = [float(r[ie] or 0), float(r[te] or 0), float(r[ss] or 0)]
        key = "other"
        if cur == fname:
            for n, lo, hi in regions:
                if lo <= int(r[0]) <= hi: key = n; break
        elif cur == "kernels.cuh":
            key = "kernels.cuh"
            acc.setdefault(key, [0, 0, 0])
        for i in range(3): acc[key][i] += v[i]; tot[i] += v[i]
for k, v in acc.items():
    print(f"{k:14s} warp-instr {v[0]:.3e} ({v[0]/tot[0]*100:5.1f}%)  thr/warp {v[1]/max(v[0],1):5.1f}  stall {v[2]/tot[2]*100:5.1f}%")
