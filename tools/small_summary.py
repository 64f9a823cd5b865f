#!/usr/bin/env python
"""Summary of bench lines written by tools/prof_small.sh (and a cfg2 bench line).
    python tools/small_summary.py gpurun_out/small_TAG_cfg1.json ..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e)
        continue
    r = d["roofline"]
    p = d.get("parity", {})
    print(f"{d['config'].get('name', f)}: {d['value'] / 1e9:.2f} G/s  step {1e3 * d['ms_per_step']:.1f} us  "
          f"kernel {1e3 * r['kernel_ms_avg']:.1f} us  {r['bound']} frac {r['frac']:.3f} "
          f"(hbm {r['hbm_frac']:.3f}, l2 {r['l2_frac']:.3f})  e2e {d['e2e']['value'] / 1e9:.2f} G/s  "
          f"flags_match {p.get('flags_match')} golden {p.get('golden_match')}")
