#!/bin/bash
# Build compile-time variants of the library on the GPU box and bench each (kernel-only
# numbers + the bench's parity sample). Usage:
#   tools/tune.sh "name1|-DSSJB_X=1 -DSSJB_Y=2" "name2|-DSSJB_X=2" -- [extra bench args]
OUT=gpurun_out; mkdir -p $OUT
VARS=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do VARS+=("$1"); shift; done
[ "$1" == "--" ] && shift
cp paper_1812_09141_b200/libssjoin_b200.so /tmp/lib_default.so
for v in "${VARS[@]}"; do
  NAME=${v%%|*}; FLAGS=${v#*|}
  rm -rf build/obj
  make -s -j16 NVFLAGS_EXTRA="$FLAGS" paper_1812_09141_b200/libssjoin_b200.so > /dev/null 2>&1 || { echo "build $NAME failed"; continue; }
  timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --join-workload none "$@" \
      > $OUT/tune_$NAME.json 2> $OUT/tune_$NAME.err
  python - "$NAME" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/tune_{v}.json"))
    r = d["roofline"]
    pa = d.get("parity", {})
    print(f"{v}: {d['config'].get('name')} {d['value']/1e9:.2f} G pairs/s, kernel {r['kernel_ms_avg']:.3f} ms, frac {r['frac']:.3f} (hbm {r.get('hbm_frac', 0):.3f}), e2e {d['e2e']['value']/1e9:.2f}, golden {pa.get('golden_match')} e2e_identical {pa.get('e2e_flags_identical')}")
except Exception as e:
    print(v, "failed", e, open(f"gpurun_out/tune_{v}.err").read()[-500:])
PY
done
cp /tmp/lib_default.so paper_1812_09141_b200/libssjoin_b200.so
