timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_filter.py -x -q > gpurun_out/t1_pytest.log 2>&1; tail -2 gpurun_out/t1_pytest.log
for W in cfg2_095 cfg2_090 cfg3; do bash tools/tune.sh "tg_$W|" "notg_$W|-DSSJB_RUN_TAGMAP=0" -- --workload $W; done
