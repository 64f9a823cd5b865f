timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t1_pytest.log 2>&1; tail -2 gpurun_out/t1_pytest.log
for W in cfg2_095 cfg2_090 cfg2; do bash tools/tune.sh "pk_$W|" -- --workload $W; done
