# round-2 evidence: bench lines (config 4, config 5 at n = 33), launch lists of
# the same commands, full capture of one config-4 batch, companions, config-5
# group-mode shape, next rows, small configs.  Each profiler run follows a
# clean run of the same command; numbers under ncu are never bench values.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_n1.json 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench_n1.json | cut -c1-200
timeout 900 python bench.py --workload cfg5 --steps 2 --warmup 1 > gpurun_out/bench_cfg5_n33.json 2> gpurun_out/bench_cfg5.err; echo bench5=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch5.log 2>&1; echo launches5=$?
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:lqj -c 30 -o /tmp/lqj_batch python tools/prof_cfg4.py > gpurun_out/ncu_cfg4.log 2>&1; echo full=$?
ncu -i /tmp/lqj_batch.ncu-rep --page raw --csv > gpurun_out/cfg4_batch.raw.csv 2>/dev/null
ncu -i /tmp/lqj_batch.ncu-rep --page source --csv --print-source sass -k regex:lqj --launch-skip 2 --launch-count 1 > gpurun_out/cfg4_p2_sass.csv 2>/dev/null
timeout 900 python tools/companions.py > gpurun_out/companions_n30.jsonl 2> gpurun_out/companions.err; echo comp=$?
timeout 900 python tools/cfg5_group.py > gpurun_out/cfg5_group_n30.jsonl 2> gpurun_out/cfg5_group.err; echo cfg5g=$?
timeout 900 python tools/next_rows.py > gpurun_out/next_rows.jsonl 2> gpurun_out/next_rows.err; echo next=$?
timeout 600 python tools/small_configs.py > gpurun_out/small_configs.jsonl 2> gpurun_out/small.err; echo small=$?
du -sh gpurun_out
