# launch lists of the two bench commands (each after a clean run of the same command); numbers under ncu are never bench values
mkdir -p gpurun_out
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo clean=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 600 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo clean5=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch5.log 2>&1; echo launches5=$?
