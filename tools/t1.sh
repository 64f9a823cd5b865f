tail -2 gpurun_out/t1_pytest.log
for i in 1 2; do bash tools/tune.sh "ds${i}_cfg3|" "nods${i}_cfg3|-DSSJB_TILE_DESC_SHFL=0" -- --workload cfg3; done
