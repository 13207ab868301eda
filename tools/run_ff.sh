mkdir -p gpurun_out
for i in 1 2; do
LQ_JIT_RUNTIME_CIRC=1 KS=11 timeout 900 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/runtime /"
KS=11 timeout 900 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed "s/^/ct /"
done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
