#!/bin/bash
# Build compile-time variants on the GPU box and time the all-GPU join of a workload with each.
#   tools/tune_join.sh "name1|-DSSJB_X=1" "name2|-DSSJB_X=0" -- [gpu_join_once.py args]
OUT=gpurun_out; mkdir -p $OUT
VARS=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do VARS+=("$1"); shift; done
[ "$1" == "--" ] && shift
cp paper_1812_09141_b200/libssjoin_b200.so /tmp/lib_default.so
for v in "${VARS[@]}"; do
  NAME=${v%%|*}; FLAGS=${v#*|}
  rm -rf build/obj
  make -s -j16 NVFLAGS_EXTRA="$FLAGS" paper_1812_09141_b200/libssjoin_b200.so > /dev/null 2>&1 || { echo "build $NAME failed"; continue; }
  for ALG in 0 1 2; do
    echo -n "$NAME alg$ALG: "
    timeout 300 python tools/gpu_join_once.py --alg $ALG --reps 3 "$@" 2> $OUT/tunej_${NAME}_$ALG.err | tail -1
  done
done
cp /tmp/lib_default.so paper_1812_09141_b200/libssjoin_b200.so
