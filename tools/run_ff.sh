mkdir -p gpurun_out
KS=11 timeout 900 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/base /"
LQ_JIT_EXTRA_OPTS=-extra-device-vectorization KS=11 timeout 900 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/edv /"
LQ_JIT_EXTRA_OPTS=--maxrregcount=160 KS=11 timeout 900 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/r160 /"
LQ_JIT_EXTRA_OPTS=-Xptxas=-O2 KS=11 timeout 900 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/O2 /"
LQ_JIT_EXTRA_OPTS=--ftz=true KS=11 timeout 900 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/ftz /"
KS=11 timeout 900 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/base /"
