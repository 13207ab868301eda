# sharded-state GPU tests on the build with balanced QFT runs in plan_circuit, then the group-mode A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "shard or group or qft or fullsize or roundtrip" > gpurun_out/gpu_tests_sharded.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests_sharded.log
tail -3 gpurun_out/gpu_tests_sharded.log
for cfg in "29 2" "29 8" "31 2" "31 8" "32 4"; do
  set -- $cfg
  AB_N=$1 AB_G=$2 timeout 1200 python tools/ab_qft_group.py balanced greedy:LQ_QFT_GREEDY=1 >> gpurun_out/ab_qft_group_balance.jsonl
done
cat gpurun_out/ab_qft_group_balance.jsonl | cut -c1-220
