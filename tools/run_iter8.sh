mkdir -p gpurun_out
R=30 python tools/small_configs.py > gpurun_out/small_configs.jsonl 2>&1; cat gpurun_out/small_configs.jsonl | cut -c1-200
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
