mkdir -p gpurun_out
for co in 3 4 3; do
CO=$co KS=11 timeout 900 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/co=$co /"
done
