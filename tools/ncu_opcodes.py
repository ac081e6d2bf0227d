#!/usr/bin/env python
"""Executed-instruction histogram by SASS opcode from an ncu report.
usage: ncu_opcodes.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if len(r) > 5 and r[0] == "Address")
ie = hdr.index("Instructions Executed"); te = hdr.index("Thread Instructions Executed"); src = hdr.index("Source")
c = Counter(); ct = Counter()
for r in rows:
    if len(r) == len(hdr) and r[0].startswith("0x"):
        ins = r[src].strip()
        if ins.startswith("@"):
            ins = ins.split(None, 1)[1]
        op = ins.split()[0] if ins else "?"
        c[op] += float(r[ie] or 0); ct[op] += float(r[te] or 0)
tot = sum(c.values())
for op, v in c.most_common(top):
    print(f"{op:28s} {v/tot*100:6.2f}%  warp-instr {v:.3e}  thr/warp {ct[op]/max(v,1):5.1f}")
