#!/bin/bash
# ncu --set full of every strategy-A kernel on cfg3 (run under gpurun; one GPU)
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-c3}
for K in long_slice_kernel bitmap_kernel run_kernel warp_tile_kernel prep_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
    -o $OUT/prof_${TAG}_$K -f python bench.py --workload cfg3 --steps 1 --warmup 1 --e2e-steps 1 \
    --no-cpu-baseline --join-workload none > $OUT/ncu_${TAG}_$K.log 2>&1
  echo "$K rc=$?"
done
