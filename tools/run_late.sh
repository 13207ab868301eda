KS=11 timeout 600 python tools/sb_probe.py cfg4 qft 2>&1 | grep -E "SB|rror"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests.log
