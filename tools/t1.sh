for W in cfg1 cfg3 cfg4; do bash tools/tune.sh "bc8_$W|" "bc4_$W|-DSSJB_BITMAP_CTAS_PER_SM=4" "bc2_$W|-DSSJB_BITMAP_CTAS_PER_SM=2" -- --workload $W; done
