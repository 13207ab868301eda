mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "qft or QFT or config2 or config1" > gpurun_out/qft_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/qft_tests.log
KS="0 11" timeout 600 python tools/qft_probe.py 2>&1 | grep -v "^$" | head
