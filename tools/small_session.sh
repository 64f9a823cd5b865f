bash tools/prof_small.sh r2a cfg1 cfg3 cfg4
OUT=gpurun_out
for K in "warp_tile_cfg3 cfg3 warp_tile_kernel" "warp_tile_cfg1 cfg1 warp_tile_kernel" "prep_cfg3 cfg3 prep_kernel"; do
  set -- $K
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
    -o $OUT/prof_k2_$1 -f python bench.py --workload $2 --steps 1 --warmup 1 --e2e-steps 1 \
    --no-cpu-baseline --join-workload none > $OUT/ncu_k2_$1.log 2>&1
  echo "$1 rc=$?"
done
