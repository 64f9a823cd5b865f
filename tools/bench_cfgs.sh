#!/bin/bash
# Quick kernel-only numbers for a list of workloads (no CPU baseline).
# Usage: tools/bench_cfgs.sh tag cfg1 cfg3 ...
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for W in "$@"; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --e2e-steps 1 --cpu-sample 2e6 > $OUT/q_${TAG}_$W.json 2> $OUT/q_${TAG}_$W.err
  python - $TAG $W <<'PY'
import json, sys
t, w = sys.argv[1:]
try:
    d = json.load(open(f"gpurun_out/q_{t}_{w}.json")); r = d["roofline"]
    print(f"{w}: {d['value']/1e9:.2f} G pairs/s, kernel {r['kernel_ms_avg']:.3f} ms, frac {r['frac']:.3f}, e2e {d['e2e']['value']/1e9:.2f}, parity {d.get('parity_sample')}")
except Exception as e:
    print(w, "failed", e, open(f"gpurun_out/q_{t}_{w}.err").read()[-800:])
PY
done
