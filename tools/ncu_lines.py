#!/usr/bin/env python
"""Top CUDA source lines of an ncu report by warp-stall samples (read here, needs -lineinfo).
    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, res, ws, ie = None, [], None, None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        ws = h.index("Warp Stall Sampling (All Samples)")
        ie = h.index("Instructions Executed")
        continue
    if ws is not None and len(r) > ws and r[0].isdigit():
        # metric columns counted from the right (source text may break the CSV quoting)
        a, b = r[len(r) - (len(h) - ws)], r[len(r) - (len(h) - ie)]
        s = int(a) if a.isdigit() else 0
        i = int(b) if b.isdigit() else 0
        if s or i:
            res.append((s, i, fname, int(r[0]), r[1].strip()))
ts = sum(x[0] for x in res) or 1
ti = sum(x[1] for x in res) or 1
print(f"samples {ts} warp-instructions {ti}")
for s, i, f, ln, src in sorted(res, reverse=True)[:N]:
    print(f"{100 * s / ts:5.1f}% stall {100 * i / ti:5.1f}% inst  {f}:{ln}  {src[:90]}")
