#!/bin/bash
# ncu --set full captures of every strategy-A kernel on the workload where it dominates, plus
# the device candidate generator (run under gpurun; one GPU). Outputs gpurun_out/prof_k_*.ncu-rep
OUT=gpurun_out; mkdir -p $OUT
cap() {  # name workload kernel-regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 \
    -o $OUT/prof_k_$1 -f python bench.py --workload $2 --steps 1 --warmup 1 --e2e-steps 1 \
    --no-cpu-baseline --join-workload none > $OUT/ncu_k_$1.log 2>&1
  echo "$1 rc=$?"
}
cap run_cfg2 cfg2 run_kernel 1
cap warp_tile_cfg3 cfg3 warp_tile_kernel 1
cap long_cfg4 cfg4 long_slice_kernel 1
cap warp_tile_cfg1 cfg1 warp_tile_kernel 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:generate_kernel -s 2 -c 1 \
  -o $OUT/prof_k_generate_cfg5 -f python tools/gpu_join_once.py --reps 1 > $OUT/ncu_k_gen.log 2>&1
echo "generate rc=$?"
