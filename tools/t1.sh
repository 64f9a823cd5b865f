tail -3 gpurun_out/t1_pytest.log
for W in cfg2 cfg3; do
bash tools/tune.sh "fk2_$W|" -- --workload $W
done
