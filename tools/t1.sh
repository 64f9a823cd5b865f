timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_filter.py -x -q > gpurun_out/t1_pytest.log 2>&1; tail -2 gpurun_out/t1_pytest.log
for W in cfg1 cfg2; do bash tools/tune.sh "ord_$W|" -- --workload $W; done
