# do two 128-byte halves of a 256-byte segment, loaded by the two CTAs of a cluster in lockstep, stream like 256-byte runs?
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tpbw tools/tile_pattern_bw.cu || exit 1
M30="0x3fe00007 0x1ff007 0xfff"
M26="0xff0007 0x3fc0007 0x7f8007 0x7ff"
for pair in 0 1 2; do
  TPBW_PAIR=$pair /tmp/tpbw masks 30 $M30 | sed "s/^{/{\"pair\": $pair, /" >> gpurun_out/tile_pattern_bw_pair.jsonl
  TPBW_PAIR=$pair /tmp/tpbw masks 26 $M26 | sed "s/^{/{\"pair\": $pair, /" >> gpurun_out/tile_pattern_bw_pair.jsonl
done
cat gpurun_out/tile_pattern_bw_pair.jsonl
