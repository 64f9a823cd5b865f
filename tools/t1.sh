bash tools/tune.sh "p1m3_cfg2|" "p1m2_cfg2|-DSSJB_RUN_MAP_BUFS=2" "p0m3_cfg2|-DSSJB_RUN_PIPE=0" "p0m2_cfg2|-DSSJB_RUN_PIPE=0 -DSSJB_RUN_MAP_BUFS=2" -- --workload cfg2
bash tools/tune.sh "p1m3_cfg5|" "p1m2_cfg5|-DSSJB_RUN_MAP_BUFS=2" -- --workload cfg5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t1_pytest.log 2>&1; tail -2 gpurun_out/t1_pytest.log
timeout 600 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py::test_trailing_uncovered_slots -q -p no:cacheprovider > gpurun_out/t1_initcheck.log 2>&1; grep "ERROR SUMMARY" gpurun_out/t1_initcheck.log; tail -1 gpurun_out/t1_initcheck.log
