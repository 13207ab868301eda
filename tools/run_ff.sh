mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "compile_time_circuit or support" 2>&1 | tail -3
