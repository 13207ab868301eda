mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.json | cut -c1-400
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q -k n32 > gpurun_out/sharded32.log 2>&1; echo sharded32=$?
tail -5 gpurun_out/sharded32.log
