# ncu captures of the n=28 companion kernels (QFT passes, XYZ expectation passes, init_random) -> csv summaries
mkdir -p gpurun_out
KS=11 timeout 600 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror"
KS=11 timeout 600 python tools/sb_probe.py cfg4 2>&1 | grep -E "probe|rror"
for m in qft expv init; do
  timeout 900 ncu -f --set full --clock-control none -k regex:'lqj|k_random|k_tile' -o /tmp/comp_$m python tools/prof_comp.py $m > gpurun_out/ncu_comp_$m.log 2>&1; echo $m=$?
  ncu -i /tmp/comp_$m.ncu-rep --page raw --csv > gpurun_out/comp_$m.raw.csv 2>/dev/null
done
du -sh gpurun_out
