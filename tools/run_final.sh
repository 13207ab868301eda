# round evidence refresh: tests, bench, launch list, full ncu capture of one batch, companions, next rows, config-5 shape
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:lqj -c 30 -o /tmp/lqj_batch python tools/prof_cfg4.py > gpurun_out/ncu_cfg4.log 2>&1; echo full=$?
ncu -i /tmp/lqj_batch.ncu-rep --page raw --csv > gpurun_out/cfg4_batch.raw.csv 2>/dev/null
ncu -i /tmp/lqj_batch.ncu-rep --page source --csv --print-source sass -k regex:lqj --launch-skip 2 --launch-count 1 > gpurun_out/cfg4_p2_sass.csv 2>/dev/null
timeout 900 python tools/companions.py > gpurun_out/companions.log 2>&1; echo comp=$?
timeout 900 python tools/next_rows.py > gpurun_out/next_rows.jsonl 2> gpurun_out/next_rows.err; echo next=$?
timeout 900 python tools/cfg5_group.py > gpurun_out/cfg5_group_n30.jsonl 2> gpurun_out/cfg5_group.err; echo cfg5g=$?
du -sh gpurun_out
