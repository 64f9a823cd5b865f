#!/usr/bin/env python
"""Instruction-count breakdown of an ncu report by straight-line SASS block (read here).
    python tools/ncu_blocks.py rep.ncu-rep units [min_share]
units = work units of the launch (e.g. candidate pairs): prints warp-instructions per unit."""
import csv, io, subprocess, sys
rep, units = sys.argv[1], float(sys.argv[2])
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ai, si, ie, ws = (h.index(k) for k in ("Address", "Source", "Instructions Executed",
                                       "Warp Stall Sampling (All Samples)"))
data = [(int(r[ai], 16) & 0xfffff, r[si].strip(), int(r[ie] or 0), int(r[ws] or 0))
        for r in rows[2:] if len(r) > ie]
tot = sum(d[2] for d in data); tots = sum(d[3] for d in data)
blocks, cur = [], None
for a, src, n, s in data:
    if cur and n == cur["n"]:
        cur["end"] = a; cur["cnt"] += 1; cur["s"] += s; cur["srcs"].append(src)
    else:
        if cur: blocks.append(cur)
        cur = {"start": a, "end": a, "n": n, "cnt": 1, "s": s, "srcs": [src]}
blocks.append(cur)
print(f"total warp-inst/unit {tot/units:.3f}")
for b in blocks:
    share = b["n"] * b["cnt"] / tot
    if share >= mn:
        ops = {}
        for x in b["srcs"]:
            op = x.split()[0] if not x.startswith("@") else x.split()[1]
            op = op.split(".")[0]
            ops[op] = ops.get(op, 0) + 1
        top = ",".join(f"{k}{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
        print(f"{b['start']:05x}-{b['end']:05x} n{b['cnt']:4d} x{b['n']/units:7.4f}/u "
              f"share {100*share:5.1f}% stall {100*b['s']/tots:5.1f}%  {top}")
