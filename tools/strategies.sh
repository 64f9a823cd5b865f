#!/bin/bash
# The paper's thread-allocation alternatives on each BASELINE config (kernel-only, parity
# sample against the reference): A (thread per pair: runs / warp tiles / long pass),
# B (CTA per probe slice, group = threads per CTA), C (G lanes per pair over merge-path
# partitions). Output: gpurun_out/strategies_<tag>.jsonl
TAG=${1:-x}
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/strategies_$TAG.jsonl
for W in ${WORKLOADS:-cfg1 cfg2 cfg3 cfg4}; do
  for S in "A 32" "B 128" "B 256" "C 4" "C 8" "C 32"; do
    set -- $S
    timeout 600 python bench.py --workload $W --strategy $1 --group $2 --steps 5 --warmup 3 \
        --e2e-steps 1 --no-cpu-baseline --join-workload none > $OUT/st_${TAG}.json 2> $OUT/st_${TAG}.err
    python - $W $1 $2 $TAG <<'PY' | tee -a $OUT/strategies_$TAG.jsonl
import json, sys
w, s, g, t = sys.argv[1:]
try:
    d = json.load(open(f"gpurun_out/st_{t}.json")); r = d["roofline"]
    print(json.dumps({"workload": w, "strategy": s, "group": int(g), "pairs_per_s": d["value"],
                      "kernel_ms": r["kernel_ms_avg"], "frac": r["frac"],
                      "golden_match": d.get("parity", {}).get("golden_match"),
                      "arm": d.get("arm")}))
except Exception as e:
    print(json.dumps({"workload": w, "strategy": s, "group": int(g), "failed": str(e)}))
PY
  done
done
