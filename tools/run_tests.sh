mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${1:-} > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -15 gpurun_out/gpu_tests.log
