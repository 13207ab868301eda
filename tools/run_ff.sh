mkdir -p gpurun_out
for i in 1 2; do
KS=11 timeout 600 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/ctab /"
LQ_JIT_NO_CTAB=1 KS=11 timeout 600 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/smemtab /"
done
