#!/usr/bin/env python
"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
    python tools/launch_table.py gpurun_out/launches_x.csv [--per-launch]"""
import collections, csv, sys

for f in [a for a in sys.argv[1:] if not a.startswith("--")]:
    rows = list(csv.reader(open(f)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    seq = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1, "ms": 1e3}.get(r[ui], 1e-3)
        k = r[ki].split("(")[0].replace("ssjb::<unnamed>::", "")[:60]
        agg[k][0] += 1
        agg[k][1] += v
        seq.append((k, v))
    tot = sum(x[1] for x in agg.values())
    print(f"{f}: {len(seq)} launches, {tot:.1f} us")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
        print(f"  {t:10.1f} us {n:5d} x  avg {t / n:8.1f} us  {k}")
    if "--per-launch" in sys.argv:
        for k, v in seq:
            print(f"    {v:9.1f} us  {k}")
