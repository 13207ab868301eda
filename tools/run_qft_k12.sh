# QFT sizes where 11- and 12-bit tiles make the same number of passes: automatic tile size (11 bits, 3 CTAs/SM)
# against 12 bits (1 CTA/SM, longer coalescing runs under the balanced packing)
mkdir -p gpurun_out
for n in ${NS:-31 32 33}; do
  AB_N=$n AB_REPS=${REPS:-4} AB_ROUNDS=2 timeout 900 python tools/ab_qft.py auto k12:AB_TILE_BITS=12 | sed "s/^{/{\"n\": $n, /" >> gpurun_out/ab_qft_k12.jsonl
done
cat gpurun_out/ab_qft_k12.jsonl | cut -c1-200
