# quick check: GPU tests, then the config-4 / QFT probe
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
KS=11 timeout 600 python tools/sb_probe.py cfg4 qft 2>&1 | grep -E "probe|rror"
