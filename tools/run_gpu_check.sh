mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 2 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | cut -c1-300
