mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
KS=11 timeout 600 python tools/jit_probe2.py 2>&1 | tail -2
