#!/usr/bin/env python
"""SASS lines of an ncu report ordered by address with executed warp-instructions (read here).
    python tools/ncu_sass_inst.py gpurun_out/prof.ncu-rep [min_share_pct]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ai, si, ws, ie = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                       "Instructions Executed"))
data = [r for r in rows[2:] if len(r) > ie]
tot_i = sum(int(r[ie] or 0) for r in data)
print(f"warp-instructions {tot_i}")
for r in data:
    i = int(r[ie] or 0)
    if 100 * i / tot_i >= mn:
        print(f"{r[ai][-5:]} {100*i/tot_i:5.2f}% {int(r[ws] or 0):6d} {r[si].strip()[:90]}")
