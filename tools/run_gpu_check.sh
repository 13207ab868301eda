mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 400 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | cut -c1-400
LQ_PROF_LAYERS=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 10 -c 1 -o gpurun_out/k_tile python tools/prof_cfg4.py > gpurun_out/ncu.log 2>&1; echo ncu=$?
