#!/bin/bash
# Every BASELINE config (kernel-only + e2e + CPU reference lines) and the end-to-end join
# (cfg5 through run_join vs the reference run_join). Output: gpurun_out/configs_<tag>.jsonl
TAG=${1:-x}
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/configs_$TAG.jsonl
for W in cfg1 cfg2 cfg2_085 cfg2_090 cfg2_095 cfg3 cfg4 cfg5; do
  J=none; [ $W == cfg2 ] && J=cfg5
  timeout 900 python bench.py --workload $W --steps 10 --warmup 3 --e2e-steps 5 --join-workload $J \
      >> $OUT/configs_$TAG.jsonl 2> $OUT/configs_${TAG}_$W.err || echo "{\"workload\": \"$W\", \"failed\": true}" >> $OUT/configs_$TAG.jsonl
done
timeout 1200 python tools/join_e2e.py --workload cfg5 > $OUT/join_e2e_$TAG.json 2> $OUT/join_e2e_$TAG.err
echo "bench_all done"
