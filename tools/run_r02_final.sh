# final round-2 refresh: all GPU tests, tools/run_r02.sh, a full capture of the
# three QFT(28) passes (balanced packing), the 13-bit QFT(30) tile-set ceilings
bash tools/run_tests.sh
bash tools/run_r02.sh
LQ_COMP_N=28 timeout 600 python tools/prof_comp.py qft > /dev/null 2>&1 && \
LQ_COMP_N=28 timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:lqj -c 3 -o /tmp/qft28 python tools/prof_comp.py qft > gpurun_out/ncu_qft28.log 2>&1; echo qft28=$?
ncu -i /tmp/qft28.ncu-rep --page raw --csv > gpurun_out/qft28.raw.csv 2>/dev/null
python tools/ncu_comp_summary.py qft28 gpurun_out/qft28.raw.csv > gpurun_out/ncu_qft28_summary.txt 2>&1
cat gpurun_out/ncu_qft28_summary.txt | cut -c1-250
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tpbw tools/tile_pattern_bw.cu && \
  /tmp/tpbw masks 30 0x3fe00007 0x1ff007 0xfff 0x3fe0000f 0x1ff00f 0x1fff > gpurun_out/tile_pattern_bw_qft30_k13.jsonl
/tmp/tpbw masks 28 0xff0000f 0xff00f 0xfff 0xff80007 0x7fc007 >> gpurun_out/tile_pattern_bw_qft30_k13.jsonl
cat gpurun_out/tile_pattern_bw_qft30_k13.jsonl
