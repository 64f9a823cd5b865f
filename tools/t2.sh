timeout 600 ncu --set full --clock-control none --import-source on -k regex:run_kernel -s 1 -c 1 \
     -o gpurun_out/prof_j95c -f python bench.py --workload cfg2_095 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline \
     --join-workload none > gpurun_out/ncu_j95c.log 2>&1; echo ncu rc=$?
