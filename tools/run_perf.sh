for b in 0 400 300 250; do LQ_BUDGET=$b KS=11 timeout 600 python tools/jit_probe2.py 2>&1 | grep "K="; done
