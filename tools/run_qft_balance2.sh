# A/B: stages of the contiguous QFT pass (LQ_QFT_CT = coalescing bits the strided passes aim for)
mkdir -p gpurun_out
for n in 25 27 31 32 33; do
  AB_N=$n AB_REPS=4 AB_ROUNDS=2 timeout 900 python tools/ab_qft.py balanced ct4:LQ_QFT_CT=4 ct5:LQ_QFT_CT=5 | sed "s/^{/{\"n\": $n, /" >> gpurun_out/ab_qft_balance2.jsonl
done
cat gpurun_out/ab_qft_balance2.jsonl | cut -c1-200
