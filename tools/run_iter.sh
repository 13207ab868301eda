# iteration check: GPU tests, then standalone-call and config-4 timings
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
python tools/host_probe.py 2>&1 | tail -5
python tools/rb_probe.py cfg4 2>&1 | grep -E "RB|Error|error" | head
