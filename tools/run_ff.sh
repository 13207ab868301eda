mkdir -p gpurun_out
timeout 900 python tools/small_configs.py > gpurun_out/small_configs.jsonl 2> gpurun_out/small_configs.err; echo small=$?
cat gpurun_out/small_configs.jsonl | cut -c1-200
