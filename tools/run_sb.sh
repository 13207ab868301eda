python tools/sb_probe.py qft 2>&1 | grep SB
LQ_SINGLEBUF=1 python tools/sb_probe.py qft 2>&1 | grep -E "SB|rror"
KS="12" LQ_SINGLEBUF=1 python tools/sb_probe.py cfg4 2>&1 | grep -E "SB|rror"
KS="12 11" python tools/sb_probe.py cfg4 2>&1 | grep -E "SB|rror"
LQ_SINGLEBUF=1 timeout 600 python -m pytest tests/test_gpu_jit.py -x -q 2>&1 | tail -2
