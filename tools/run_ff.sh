mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "support_restriction or xyz_ring or config3 or app_e or cry or config4" 2>&1 | tail -3
for i in 1 2; do
LQ_NO_SUPPORT=1 KS=11 timeout 600 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed 's/^/nosupport /'
KS=11 timeout 600 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror" | sed 's/^/support /'
done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
