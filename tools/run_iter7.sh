mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python tools/next_rows.py > gpurun_out/next_rows.jsonl 2> gpurun_out/next_rows.err; echo next=$?
cut -c1-300 gpurun_out/next_rows.jsonl
KS=11 timeout 600 python tools/sb_probe.py cfg4 2>&1 | grep -E "SB|rror"
