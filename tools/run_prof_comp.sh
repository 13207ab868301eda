mkdir -p gpurun_out
for m in qft expv init; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'lqj|k_random|k_tile' -o /tmp/comp_$m python tools/prof_comp.py $m > gpurun_out/ncu_comp_$m.log 2>&1; echo $m=$?
  ncu -i /tmp/comp_$m.ncu-rep --page raw --csv > gpurun_out/comp_$m.raw.csv 2>/dev/null
  ncu -i /tmp/comp_$m.ncu-rep --page details --csv > gpurun_out/comp_$m.details.csv 2>/dev/null
done
ls -la /tmp/*.ncu-rep
cp /tmp/comp_qft.ncu-rep gpurun_out/ 2>/dev/null
du -sh gpurun_out
