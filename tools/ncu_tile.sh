#!/bin/bash
# ncu capture of the dominant kernel (tile_kernel) for one bench step, plus the launch list.
TAG=${1:-x}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-run_kernel} -s ${KSKIP:-1} -c 1 \
   -o $OUT/prof_$TAG -f python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline "${@:2}" \
   > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
