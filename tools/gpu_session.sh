#!/bin/bash
# One GPU session (run under gpurun): tests, bench, ncu launch list + full capture.
# Usage: tools/gpu_session.sh [tag]   env: SKIP_TESTS=1 SKIP_NCU=1 STEPS=n KREGEX=... BENCH_ARGS=...
set -u
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
nproc >> $OUT/gpu_$TAG.txt
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
  tail -3 $OUT/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:-} > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
echo "bench rc=$?"; cat $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 \
     --no-cpu-baseline --join-workload none > $OUT/ncu_launch_bench_$TAG.log 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-run_kernel} -s ${KSKIP:-1} -c 1 \
     -o $OUT/prof_$TAG -f python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline \
     --join-workload none > $OUT/ncu_full_$TAG.log 2>&1
  echo "ncu full rc=$?"
fi
