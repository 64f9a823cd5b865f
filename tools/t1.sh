timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t1_pytest.log 2>&1; tail -2 gpurun_out/t1_pytest.log
bash tools/tune.sh "cl_cfg2|" -- --workload cfg2
