mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
KS=11 timeout 600 python tools/jit_probe2.py 2>&1 | tail -2
LQ_PROF_LAYERS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:lqj -s 4 -c 1 -o gpurun_out/lqj4 python tools/prof_cfg4.py > gpurun_out/ncu5.log 2>&1; echo ncu=$?
