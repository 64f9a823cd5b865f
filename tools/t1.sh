timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t1_pytest.log 2>&1; tail -2 gpurun_out/t1_pytest.log
for W in cfg3 cfg1; do
bash tools/tune.sh "ub_$W|" -- --workload $W
done
