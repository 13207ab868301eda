for cb in 2 1; do LQ_COALESCE=$cb KS=11,12 timeout 600 python tools/jit_probe2.py 2>&1 | grep "K="; done
