# the automatic 12-bit rule of plan_qft (same pass count, spare coalescing bit): QFT tests, A/B against LQ_QFT_K11=1, config-5 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "qft or fullsize or n33 or config5 or cfg5" > gpurun_out/gpu_tests_qft_k12.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests_qft_k12.log
tail -3 gpurun_out/gpu_tests_qft_k12.log
for n in 26 27 33; do
  AB_N=$n AB_REPS=5 AB_ROUNDS=2 timeout 900 python tools/ab_qft.py rule k11:LQ_QFT_K11=1 | sed "s/^{/{\"n\": $n, /" >> gpurun_out/ab_qft_k12_rule.jsonl
done
cat gpurun_out/ab_qft_k12_rule.jsonl | cut -c1-200
timeout 900 python bench.py --workload cfg5 --steps 2 --warmup 1 > gpurun_out/bench_cfg5_k12.json 2> gpurun_out/bench_cfg5_k12.err; echo bench5=$?
tail -1 gpurun_out/bench_cfg5_k12.json | cut -c1-300
