for W in cfg3 cfg1; do bash tools/tune.sh "mb8_$W|" "mb6_$W|-DSSJB_TILE_MIN_BLOCKS=6" "mb7_$W|-DSSJB_TILE_MIN_BLOCKS=7" -- --workload $W; done
