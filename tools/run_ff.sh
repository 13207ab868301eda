mkdir -p gpurun_out
for b in 4 2 3 4; do
LQ_PSR_BATCH=$b KS=11 timeout 900 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/B=$b /"
done
