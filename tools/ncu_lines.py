#!/usr/bin/env python
"""Aggregate an ncu report's source page by (file, CUDA source line) (needs
-lineinfo and --import-source on).  usage: ncu_lines.py report.ncu-rep [top_n]"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if len(r) > 5 and r[0] == "Line No")
ie = hdr.index("Instructions Executed")
te = hdr.index("Thread Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
lines = []
cur_file = "?"
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = os.path.basename(r[1])
        continue
    if len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
        try:
            lines.append((float(r[ie] or 0), float(r[te] or 0), float(r[ss] or 0), f"{cur_file}:{r[0]}", r[1].strip()))
        except ValueError:
            pass
T = [sum(x[i] for x in lines) for i in range(3)]
print(f"total warp-instr {T[0]:.3e}  thread-instr {T[1]:.3e}  stall samples {T[2]:.0f}")
for v in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{v[0]/T[0]*100:6.2f}% instr {v[1]/max(v[0],1):5.1f}thr {v[2]/max(T[2],1)*100:6.2f}%stall  {v[3]}: {v[4][:80]}")
