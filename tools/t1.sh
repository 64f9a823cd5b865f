timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_filter.py tests/test_gpu_pipeline.py tests/test_gpu_multi.py -x -q > gpurun_out/t1_pytest.log 2>&1; tail -2 gpurun_out/t1_pytest.log
for W in cfg2 cfg2_095 cfg2_090 cfg2_085; do bash tools/tune.sh "q_$W|" -- --workload $W; done
