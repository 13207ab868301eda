mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/san_$tool.log 2>&1; echo $tool=$?
tail -3 gpurun_out/san_$tool.log
done
