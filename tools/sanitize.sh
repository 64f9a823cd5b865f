#!/bin/bash
# compute-sanitizer over a representative subset of the GPU parity tests (run under gpurun).
# Every kernel family runs: prep/bitmap, run_kernel, warp_tile_kernel, long_slice_kernel
# (strategy A), block_kernel (B), path_kernel (C), pairs/sort, the GPU filter kernels and the
# multi-device path. Usage: tools/sanitize.sh tag [tools...]
TAG=${1:-r2}; shift
OUT=gpurun_out; mkdir -p $OUT
SEL="tests/test_gpu_parity.py::test_golden_chunks_all_strategies tests/test_gpu_parity.py::test_random_chunks_vs_oracle tests/test_gpu_parity.py::test_long_sets_bitmaps_and_deferral tests/test_gpu_parity.py::test_trailing_uncovered_slots tests/test_gpu_parity.py::test_empty_and_tiny tests/test_gpu_parity.py::test_token_value_ranges tests/test_gpu_parity.py::test_gpu_pair_decoding tests/test_gpu_filter.py::test_gpu_join_matches_brute_force tests/test_gpu_multi.py::test_multi_random_vs_oracle"
TOOLS=("$@"); [ ${#TOOLS[@]} -eq 0 ] && TOOLS=(memcheck racecheck synccheck initcheck)
for T in "${TOOLS[@]}"; do
  timeout 2400 compute-sanitizer --tool $T --target-processes all --print-limit 100 \
     --log-file $OUT/sanitizer_${TAG}_${T}.log \
     python -m pytest $SEL -q -x -p no:cacheprovider > $OUT/sanitizer_${TAG}_${T}.out 2>&1
  echo "$T rc=$? $(tail -n 1 $OUT/sanitizer_${TAG}_${T}.out)"
  grep -h "ERROR SUMMARY\|RACECHECK SUMMARY" $OUT/sanitizer_${TAG}_${T}.log | sort | uniq -c | head -5
done
