# round-1 evidence: bench line, launch list of the same command, full capture of one batch's passes
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lqj -c 30 -o gpurun_out/lqj_batch python tools/prof_cfg4.py > gpurun_out/ncu_full.log 2>&1; echo full=$?
