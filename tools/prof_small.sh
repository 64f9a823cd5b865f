#!/bin/bash
# Small-chunk configs (cfg1, cfg3, cfg4): kernel-only bench lines + per-kernel launch lists.
# Usage (under gpurun): tools/prof_small.sh tag [workloads...]
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for W in "${@:-cfg1 cfg3 cfg4}"; do
  timeout 600 python bench.py --workload $W --steps 20 --warmup 5 --e2e-steps 3 --cpu-reps 1 \
     --join-workload none > $OUT/small_${TAG}_$W.json 2> $OUT/small_${TAG}_$W.err
  echo "$W bench rc=$?"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file $OUT/launches_small_${TAG}_$W.csv python bench.py --workload $W --steps 2 --warmup 1 \
     --e2e-steps 1 --no-cpu-baseline --join-workload none > /dev/null 2>&1
  echo "$W launches rc=$?"
done
