timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
N=30 GS=1,2,4 timeout 1200 python tools/cfg5_probe.py 2>&1 | tail -3
