#!/bin/bash
# Launch list + full ncu capture of one kernel for a given workload.
# Usage: tools/prof_cfg.sh <workload> <kernel-regex> <tag> [skip]
W=$1; K=$2; TAG=$3; SKIP=${4:-1}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $OUT/launches_$TAG.csv python bench.py --workload $W --steps 2 --warmup 1 --e2e-steps 1 \
   --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
   -o $OUT/prof_$TAG -f python bench.py --workload $W --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline \
   > $OUT/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
