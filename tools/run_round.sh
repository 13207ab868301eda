# round evidence: bench line, launch list of the same command, companions at n=30
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 python tools/companions.py > gpurun_out/companions.log 2>&1; echo comp=$?
grep -v JSON gpurun_out/companions.log | cut -c1-200
