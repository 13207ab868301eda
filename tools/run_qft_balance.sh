# same-box A/B of plan_qft's balanced stage packing against the greedy one
# (LQ_QFT_GREEDY=1), the new closed-form tests, and the access-pattern
# ceilings of a 13-bit-tile QFT(30) plan (256-byte runs) next to the 12-bit one
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "qft" > gpurun_out/gpu_tests_qft.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests_qft.log
tail -3 gpurun_out/gpu_tests_qft.log
for n in 26 28 29 30 31 33; do
  AB_N=$n AB_REPS=4 AB_ROUNDS=2 timeout 900 python tools/ab_qft.py balanced greedy:LQ_QFT_GREEDY=1 | sed "s/^{/{\"n\": $n, /" >> gpurun_out/ab_qft_balance.jsonl
done
cat gpurun_out/ab_qft_balance.jsonl | cut -c1-200
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tpbw tools/tile_pattern_bw.cu && \
  /tmp/tpbw masks 30 0x3fe00007 0x1ff007 0xfff 0x3fe0000f 0x1ff00f 0x1fff > gpurun_out/tile_pattern_bw_qft30_k13.jsonl
cat gpurun_out/tile_pattern_bw_qft30_k13.jsonl
