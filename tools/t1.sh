bash tools/tune.sh "mp32|" "mp64|-DSSJB_MAX_PIECES=64" "mp128|-DSSJB_MAX_PIECES=128" "mp32b|" "mp64b|-DSSJB_MAX_PIECES=64" -- --workload cfg2 --e2e-steps 5
