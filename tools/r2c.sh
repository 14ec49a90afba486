S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $S --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2c_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r2c_$tool.log
done
