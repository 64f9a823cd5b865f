timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_filter.py -x -q > gpurun_out/t1_pytest.log 2>&1; tail -2 gpurun_out/t1_pytest.log
for W in cfg2_085 cfg5; do
bash tools/tune.sh "def_$W|" "two_$W|-DSSJB_RUN_MB3_BELOW=0" "three_$W|-DSSJB_RUN_MB3_BELOW=1000000000" -- --workload $W
done
for W in cfg2 cfg2_090 cfg2_095 cfg3 cfg4 cfg1; do
bash tools/tune.sh "def_$W|" -- --workload $W
done
