mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -4 gpurun_out/gpu_tests.log
python tools/next_rows.py > gpurun_out/next_rows.jsonl 2>gpurun_out/next_rows.err; tail -3 gpurun_out/next_rows.err; cut -c1-250 gpurun_out/next_rows.jsonl
