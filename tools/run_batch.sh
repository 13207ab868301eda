for b in 2 4 8; do LQ_PSR_BATCH=$b KS=11 python tools/sb_probe.py cfg4 2>&1 | grep -E "SB|rror" | sed "s/^/B=$b /"; done
