# full ncu capture of the 30 tile passes of one config-4 batch (2 circuits per launch)
mkdir -p gpurun_out
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:lqj -c 30 -o /tmp/lqj_batch python tools/prof_cfg4.py > gpurun_out/ncu_cfg4.log 2>&1; echo full=$?
ncu -i /tmp/lqj_batch.ncu-rep --page raw --csv > gpurun_out/cfg4_batch.raw.csv 2>/dev/null
ncu -i /tmp/lqj_batch.ncu-rep --page source --csv --print-source sass -k regex:lqj --launch-skip 2 --launch-count 1 > gpurun_out/cfg4_p2_sass.csv 2>/dev/null
ncu -i /tmp/lqj_batch.ncu-rep --page source --csv --print-source sass -k regex:lqj --launch-skip 5 --launch-count 1 > gpurun_out/cfg4_p5_sass.csv 2>/dev/null
ls -la gpurun_out/*.csv | tail -3
