mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -4 gpurun_out/gpu_tests.log
timeout 900 python tools/companions.py > gpurun_out/companions.log 2>&1; echo comp=$?
grep -v JSON gpurun_out/companions.log | cut -c1-160
