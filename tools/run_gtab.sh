KS=11 python tools/sb_probe.py cfg4 2>&1 | grep -E "SB|rror" | sed 's/^/base /'
LQ_JIT_GTAB=1 KS=11 python tools/sb_probe.py cfg4 2>&1 | grep -E "SB|rror" | sed 's/^/gtab /'
KS=11 python tools/sb_probe.py cfg4 2>&1 | grep -E "SB|rror" | sed 's/^/base /'
LQ_JIT_GTAB=1 KS=11 python tools/sb_probe.py cfg4 2>&1 | grep -E "SB|rror" | sed 's/^/gtab /'
LQ_JIT_GTAB=1 timeout 600 python -m pytest tests/test_gpu_jit.py -x -q 2>&1 | tail -1
