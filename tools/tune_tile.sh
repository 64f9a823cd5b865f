#!/bin/bash
# Build tile-kernel geometry variants on the GPU box and bench each (kernel-only numbers).
# Usage: tools/tune_tile.sh "256:8:4 128:8:8 256:4:4" [extra bench args]
VARIANTS=${1:-"256:8:4"}
shift
OUT=gpurun_out; mkdir -p $OUT
cp paper_1812_09141_b200/libssjoin_b200.so /tmp/lib_default.so
for v in $VARIANTS; do
  IFS=: read T I B CP ES WT <<< "$v"
  CP=${CP:-64}
  ES=${ES:-0}
  WT=${WT:-1}
  rm -rf build/obj
  make -s -j16 NVFLAGS_EXTRA="-DSSJB_TILE_THREADS=$T -DSSJB_TILE_ITEMS=$I -DSSJB_TILE_MIN_BLOCKS=$B -DSSJB_TILE_BM_COPY_MIN=$CP -DSSJB_EARLY_SECTOR=$ES -DSSJB_WARP_TILES=$WT" \
       paper_1812_09141_b200/libssjoin_b200.so > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 1 --cpu-sample 4e6 "$@" \
      > $OUT/tune_$v.json 2> $OUT/tune_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/tune_{v}.json"))
    r = d["roofline"]
    print(f"{v}: {d['value']/1e9:.2f} G pairs/s, kernel {r['kernel_ms_avg']:.3f} ms, frac {r['frac']:.3f}, e2e {d['e2e']['value']/1e9:.2f}, parity {d.get('parity_sample')}")
except Exception as e:
    print(v, "failed", e)
PY
done
cp /tmp/lib_default.so paper_1812_09141_b200/libssjoin_b200.so
