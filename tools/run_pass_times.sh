python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 0 3; do
RELABEL=$r timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum --clock-control none -k regex:lqj --launch-skip 280 --launch-count 28 --csv python tools/pass_times.py > gpurun_out/pt_$r.csv 2> gpurun_out/pt_$r.err; echo r$r=$?
done
