#!/usr/bin/env python
"""Top stalled SASS lines of an ncu report with their dominant stall reasons (read here).
    python tools/ncu_hot.py gpurun_out/prof.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ai, si, ws, ie = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                       "Instructions Executed"))
sc = [(i, k) for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
data = [r for r in rows[2:] if len(r) > ie]
tot_s = sum(int(r[ws] or 0) for r in data); tot_i = sum(int(r[ie] or 0) for r in data)
print(f"samples {tot_s} warp-instructions {tot_i}")
for r in sorted(data, key=lambda r: -int(r[ws] or 0))[:N]:
    s = int(r[ws] or 0)
    why = sorted(((int(r[i] or 0), k[6:]) for i, k in sc), reverse=True)[:2]
    print(f"{100*s/tot_s:5.1f}% {100*int(r[ie] or 0)/tot_i:5.2f}%i {r[ai][-5:]} {r[si].strip()[:60]:60s} "
          + " ".join(f"{k}:{100*v/max(s,1):.0f}%" for v, k in why))
