mkdir -p gpurun_out
KS=11 timeout 600 python tools/sb_probe.py cfg4 2>&1 | grep -E "SB|rror"
timeout 600 python tools/host_probe.py 2>&1 | grep expval
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
