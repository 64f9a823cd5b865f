bash tools/tune.sh "new_cfg2|" "noreq_cfg2|-DSSJB_RUN_REQTAB=0" "nooff_cfg2|-DSSJB_RUN_MAPOFF=0" -- --workload cfg2
bash tools/tune.sh "new_cfg5|" -- --workload cfg5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t1_pytest.log 2>&1; tail -2 gpurun_out/t1_pytest.log
